"""TEST INFRASTRUCTURE — ctypes binding of the compiled reference (oracle/_ref/libvkref.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module.  The library is the reference's own C++ sources built unmodified
by oracle/Makefile (see oracle/ref_capi.cpp for the forwarded entry points).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libvkref.so")

_u64p = ctypes.POINTER(ctypes.c_uint64)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int)

# Status codes shared with include/vk_rl.h.
CODE_NAMES = {1: "Error", 2: "ShapeMismatch", 3: "NegativeInput", 4: "UnnormalizedPsf",
              5: "DegenerateReference", 6: "TooSmall", 7: "OddExtent", 11: "KernelTooLarge",
              12: "BadMagic", 13: "HeaderMismatch", 14: "TruncatedPayload", 15: "PlacementFailure",
              16: "EvenExtent", 99: "Other"}

METRICS = {"si_psnr_vs_input": 0, "ssim_vs_prev": 1, "frc_resolution": 2}


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = CODE_NAMES.get(code, "?")


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        L.vkref_good_size.restype = ctypes.c_uint64
        L.vkref_good_size.argtypes = [ctypes.c_uint64]
        L.vkref_richardson_lucy.restype = ctypes.c_int
        L.vkref_richardson_lucy.argtypes = [
            ctypes.c_int, _u64p, _f32p, ctypes.c_int, _u64p, _f32p, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f32p, _f64p, _f64p, _f64p,
            _i32p, _i32p, _u64p, ctypes.c_char_p, ctypes.c_int]
        L.vkref_rl_step.restype = ctypes.c_int
        L.vkref_rl_step.argtypes = [ctypes.c_int, _u64p, _f32p, _f32p, _u64p, _f32p, ctypes.c_int,
                                    _f32p, ctypes.c_char_p, ctypes.c_int]
        L.vkref_fft_convolve.restype = ctypes.c_int
        L.vkref_fft_convolve.argtypes = [ctypes.c_int, _u64p, _f32p, _u64p, _f32p, ctypes.c_int,
                                         _f32p, ctypes.c_char_p, ctypes.c_int]
        L.vkref_gaussian_psf.restype = ctypes.c_int
        L.vkref_gaussian_psf.argtypes = [ctypes.c_int, _u64p, _f64p, ctypes.c_int, _f32p,
                                         ctypes.c_char_p, ctypes.c_int]
        L.vkref_generate_blobs.restype = ctypes.c_int
        L.vkref_generate_blobs.argtypes = [_u64p, ctypes.c_uint64, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_uint64, ctypes.c_double,
                                           _f32p, ctypes.c_char_p, ctypes.c_int]
        L.vkref_si_psnr.restype = ctypes.c_int
        L.vkref_si_psnr.argtypes = [ctypes.c_int, _u64p, _f32p, _f32p, _f64p, ctypes.c_char_p,
                                    ctypes.c_int]
        L.vkref_single_image_frc.restype = ctypes.c_int
        L.vkref_single_image_frc.argtypes = [ctypes.c_int, _u64p, _f32p, ctypes.c_double, _f64p,
                                             ctypes.c_char_p, ctypes.c_int]
        L.vkref_ssim.restype = ctypes.c_int
        L.vkref_ssim.argtypes = [ctypes.c_int, _u64p, _f32p, _f32p, _f64p, ctypes.c_char_p,
                                 ctypes.c_int]
        L.vkref_gaussian.restype = ctypes.c_int
        L.vkref_gaussian.argtypes = [ctypes.c_int, _u64p, _f32p, ctypes.c_double, ctypes.c_double,
                                     _f32p, ctypes.c_char_p, ctypes.c_int]
        if hasattr(L, "vkref_write_volume"):
            L.vkref_write_volume.restype = ctypes.c_int
            L.vkref_write_volume.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, _u64p,
                                             ctypes.c_void_p, _f64p, ctypes.c_char_p, ctypes.c_int]
            L.vkref_read_volume.restype = ctypes.c_int
            L.vkref_read_volume.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int), _u64p,
                                            ctypes.POINTER(ctypes.c_int), _f64p, _f32p,
                                            ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int]
        _lib = L
    return _lib


def _shape(a) -> ctypes.Array:
    return (ctypes.c_uint64 * max(len(a), 1))(*[int(x) for x in a])


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_f32p)


def _check(rc: int, err) -> None:
    if rc != 0:
        raise RefError(rc, err.value.decode())


def good_size(n: int) -> int:
    return int(lib().vkref_good_size(n))


@dataclass
class RefResult:
    estimate: np.ndarray
    metric: np.ndarray
    wall_s: np.ndarray
    loglik: np.ndarray
    iters_run: int
    stop_reason: str
    fft_shape: tuple = field(default_factory=tuple)


def richardson_lucy(observed, psf, metric="si_psnr_vs_input", rel_tol=1e-3, patience=3,
                    max_iters=100, flat_init=False, accelerated=False) -> RefResult:
    obs = np.ascontiguousarray(observed, dtype=np.float32)
    k = np.ascontiguousarray(psf, dtype=np.float32)
    out = np.empty_like(obs)
    n = max(int(max_iters), 1)
    mv, ws, ll = np.zeros(n), np.zeros(n), np.zeros(n)
    iters, reason = ctypes.c_int(0), ctypes.c_int(0)
    fs = (ctypes.c_uint64 * max(obs.ndim, 1))()
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_richardson_lucy(
        obs.ndim, _shape(obs.shape), _fp(obs), k.ndim, _shape(k.shape), _fp(k), METRICS[metric],
        float(rel_tol), int(patience), int(max_iters), int(bool(flat_init)), int(bool(accelerated)),
        _fp(out), mv.ctypes.data_as(_f64p), ws.ctypes.data_as(_f64p), ll.ctypes.data_as(_f64p),
        ctypes.byref(iters), ctypes.byref(reason), fs, err, 512)
    _check(rc, err)
    it = iters.value
    return RefResult(out, mv[:it], ws[:it], ll[:it], it,
                     "converged" if reason.value == 1 else "max_iters",
                     tuple(int(fs[i]) for i in range(obs.ndim)))


def rl_step(estimate, observed, psf, accelerated=False) -> np.ndarray:
    e = np.ascontiguousarray(estimate, dtype=np.float32)
    o = np.ascontiguousarray(observed, dtype=np.float32)
    k = np.ascontiguousarray(psf, dtype=np.float32)
    out = np.empty(e.shape, np.float32)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_rl_step(e.ndim, _shape(e.shape), _fp(e), _fp(o), _shape(k.shape), _fp(k),
                             int(bool(accelerated)), _fp(out), err, 512)
    _check(rc, err)
    return out


def fft_convolve(img, kernel, circular=False) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.float32)
    k = np.ascontiguousarray(kernel, dtype=np.float32)
    out = np.empty(a.shape, np.float32)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_fft_convolve(a.ndim, _shape(a.shape), _fp(a), _shape(k.shape), _fp(k),
                                  int(bool(circular)), _fp(out), err, 512)
    _check(rc, err)
    return out


def gaussian_psf(shape, sigmas) -> np.ndarray:
    sig = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, np.float64)))
    out = np.empty(tuple(shape), np.float32)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_gaussian_psf(len(shape), _shape(shape), sig.ctypes.data_as(_f64p), sig.size,
                                  _fp(out), err, 512)
    _check(rc, err)
    return out


def generate_blobs(shape, n_objects=20, radius_min=6.0, radius_max=10.0, seed=0,
                   noise_sigma=0.05) -> np.ndarray:
    out = np.empty(tuple(shape), np.float32)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_generate_blobs(_shape(shape), n_objects, radius_min, radius_max, seed,
                                    noise_sigma, _fp(out), err, 512)
    _check(rc, err)
    return out


def si_psnr(x, ref) -> float:
    a = np.ascontiguousarray(x, dtype=np.float32)
    b = np.ascontiguousarray(ref, dtype=np.float32)
    v = ctypes.c_double(0)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_si_psnr(a.ndim, _shape(a.shape), _fp(a), _fp(b), ctypes.byref(v), err, 512)
    _check(rc, err)
    return v.value


def single_image_frc(x, spacing=1.0) -> float:
    a = np.ascontiguousarray(x, dtype=np.float32)
    v = ctypes.c_double(0)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_single_image_frc(a.ndim, _shape(a.shape), _fp(a), float(spacing),
                                      ctypes.byref(v), err, 512)
    _check(rc, err)
    return v.value


def ssim(x, ref) -> float:
    """metrics::ssim as shipped (reads freed temporaries; see ref_capi.cpp)."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    b = np.ascontiguousarray(ref, dtype=np.float32)
    v = ctypes.c_double(0)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_ssim(a.ndim, _shape(a.shape), _fp(a), _fp(b), ctypes.byref(v), err, 512)
    _check(rc, err)
    return v.value


def gaussian(x, sigma=1.5, truncate=3.5) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(a.shape, np.float32)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_gaussian(a.ndim, _shape(a.shape), _fp(a), float(sigma), float(truncate),
                              _fp(out), err, 512)
    _check(rc, err)
    return out


_ELEM = {np.dtype(np.float32): 0, np.dtype(np.uint16): 1, np.dtype(np.uint32): 2, np.dtype(np.bool_): 3}


def write_volume(path, arr, spacing=None) -> None:
    """io::write_volume (reads the reference's own bytes; needs io.cpp built)."""
    a = np.ascontiguousarray(arr)
    if a.dtype == np.bool_:
        a = a.astype(np.uint8)
        elem = 3
    else:
        elem = _ELEM[a.dtype]
    sp = None if spacing is None else np.ascontiguousarray(spacing, np.float64)
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_write_volume(str(path).encode(), elem, a.ndim, _shape(a.shape), a.ctypes.data,
                                  None if sp is None else sp.ctypes.data_as(_f64p), err, 512)
    _check(rc, err)


def read_volume(path):
    """io::read_volume -> (f32 values, elem id, spacing or None)."""
    elem, rank, has = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    shape = (ctypes.c_uint64 * 4)()
    sp = (ctypes.c_double * 4)()
    err = ctypes.create_string_buffer(512)
    rc = lib().vkref_read_volume(str(path).encode(), ctypes.byref(elem), ctypes.byref(rank), shape,
                                 ctypes.byref(has), sp, None, 0, err, 512)
    _check(rc, err)
    shp = tuple(int(shape[i]) for i in range(rank.value))
    out = np.empty(shp, np.float32)
    rc = lib().vkref_read_volume(str(path).encode(), ctypes.byref(elem), ctypes.byref(rank), shape,
                                 ctypes.byref(has), sp, _fp(out), out.size, err, 512)
    _check(rc, err)
    return out, elem.value, (tuple(sp[i] for i in range(rank.value)) if has.value else None)
