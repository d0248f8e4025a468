"""B200-native Richardson-Lucy deconvolution behind the reference's deconv API.

Python mirror of the reference's `voxelkit::deconv` interface
(/root/reference/proj/include/voxelkit/deconv.hpp:28-103) over the C ABI in
include/vk_rl.h, implemented by hand-written sm_100a CUDA kernels in
paper_2510_14143_b200/csrc (built in-tree into lib/libvkrl.so).  Same names,
argument meanings and error behaviour as the reference:

    richardson_lucy(observed, psf, rule=StoppingRule(), flat_init=False) -> RlResult
    rl_step(estimate, observed, transforms_or_psf) -> ndarray
    RlTransforms(image_shape, psf, threads=...)
    StoppingRule / StopMetric / IterationRecord / IterationTrace / RlResult
    errors: Error, ShapeMismatch, NegativeInput, UnnormalizedPsf, DegenerateReference, ...

There is no CPU fallback: importing works without a GPU, but every compute
call goes through libvkrl.so and raises if the library or a GPU is missing.
"""
from __future__ import annotations

import ctypes
import io
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VK_RL_LIB") or os.path.join(_HERE, "lib", "libvkrl.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "vk_rl.h")
HEADER_PATHS = [HEADER_PATH, os.path.join(os.path.dirname(_HERE), "include", "vk_io.h")]


# --- errors (reference: proj/include/voxelkit/errors.hpp:25-70) -------------
class Error(RuntimeError):
    """voxelkit::Error.  str(e) equals the reference's what()."""


class ShapeMismatch(Error):
    pass


class NegativeInput(Error):
    pass


class UnnormalizedPsf(Error):
    pass


class DegenerateReference(Error):
    pass


class TooSmall(Error):
    pass


class OddExtent(Error):
    pass


class CudaError(Error):
    pass


class Unsupported(Error):
    pass


class KernelTooLarge(Error):
    pass


class BadMagic(Error):
    pass


class HeaderMismatch(Error):
    pass


class TruncatedPayload(Error):
    pass


class PlacementFailure(Error):
    pass


class EvenExtent(Error):
    pass


KERNEL_KINDS = ("x_fwd", "x_ratio", "x_update", "y_fwd", "z_conv", "y_inv", "y_conv", "yz_dataflow",
                "yz_cluster")  # vk_kernel_kind

_STATUS = {1: Error, 2: ShapeMismatch, 3: NegativeInput, 4: UnnormalizedPsf, 5: DegenerateReference,
           6: TooSmall, 7: OddExtent, 8: CudaError, 9: CudaError, 10: Unsupported, 11: KernelTooLarge,
           12: BadMagic, 13: HeaderMismatch, 14: TruncatedPayload, 15: PlacementFailure, 16: EvenExtent}


# --- ctypes binding -----------------------------------------------------------
class _Rule(ctypes.Structure):
    _fields_ = [("metric", ctypes.c_int), ("rel_tol", ctypes.c_double), ("patience", ctypes.c_int),
                ("max_iters", ctypes.c_int), ("spacing", ctypes.c_double)]


_dp = ctypes.POINTER(ctypes.c_double)


class _Trace(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_int), ("metric", _dp), ("wall_s", _dp), ("log_likelihood", _dp),
                ("iters_run", ctypes.c_int), ("stop_reason", ctypes.c_int),
                ("fft_shape", ctypes.c_uint64 * 3)]


class _VolumeInfo(ctypes.Structure):
    _fields_ = [("elem", ctypes.c_int), ("rank", ctypes.c_int), ("shape", ctypes.c_uint64 * 4),
                ("has_spacing", ctypes.c_int), ("spacing", ctypes.c_double * 4),
                ("payload_offset", ctypes.c_uint64), ("payload_bytes", ctypes.c_uint64)]


class _SynthSpec(ctypes.Structure):
    _fields_ = [("shape", ctypes.c_uint64 * 3), ("n_objects", ctypes.c_uint64), ("radius_min", ctypes.c_double),
                ("radius_max", ctypes.c_double), ("seed", ctypes.c_uint64), ("noise_sigma", ctypes.c_double),
                ("anisotropy", ctypes.c_double), ("inplane_margin", ctypes.c_double)]


_u64p = ctypes.POINTER(ctypes.c_uint64)
_fp = ctypes.POINTER(ctypes.c_float)
_vp = ctypes.c_void_p
_lib = None


def lib() -> ctypes.CDLL:
    """Load lib/libvkrl.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                           "(the CUDA path is the only implementation)")
    L = ctypes.CDLL(LIB_PATH)
    i, st = ctypes.c_int, ctypes.c_int
    L.vk_rl_plan_create.argtypes = [i, i, _u64p, i, _u64p, _fp, i, ctypes.POINTER(_vp)]
    L.vk_rl_plan_shapes.argtypes = [_vp, ctypes.POINTER(i), _u64p, _u64p, _u64p]
    L.vk_rl_plan_device_bytes.argtypes = [_vp, _u64p]
    L.vk_rl_plan_launches.argtypes = [_vp, _u64p]
    L.vk_rl_plan_destroy.argtypes = [_vp]
    L.vk_rl_run.argtypes = [_vp, _vp, _vp, ctypes.POINTER(_Rule), i, ctypes.POINTER(_Trace)]
    L.vk_rl_run_device.argtypes = [_vp, _vp, _vp, ctypes.POINTER(_Rule), i, ctypes.POINTER(_Trace), _vp]
    L.vk_rl_run_batch.argtypes = [_vp, i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_Rule), i,
                                  ctypes.POINTER(_Trace)]
    L.vk_rl_run_batch_device.argtypes = [_vp, i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_Rule),
                                         i, ctypes.POINTER(_Trace), _vp]
    L.vk_rl_run_batch_device.restype = st
    L.vk_rl_plan_lanes.argtypes = [_vp, ctypes.POINTER(i)]
    L.vk_rl_plan_lanes.restype = st
    L.vk_rl_step.argtypes = [_vp, _vp, _vp, _vp]
    L.vk_rl_step_device.argtypes = [_vp, _vp, _vp, _vp, _vp]
    L.vk_richardson_lucy.argtypes = [i, i, _u64p, _vp, i, _u64p, _fp, ctypes.POINTER(_Rule), i, _vp,
                                     ctypes.POINTER(_Trace)]
    L.vk_rl_step_psf.argtypes = [i, i, _u64p, _vp, _vp, i, _u64p, _fp, _vp]
    L.vk_conv_plan_create.argtypes = [i, i, _u64p, i, _u64p, _fp, i, ctypes.POINTER(_vp)]
    L.vk_conv_run.argtypes = [_vp, _vp, _vp]
    L.vk_conv_run_device.argtypes = [_vp, _vp, _vp, _vp]
    L.vk_fft_convolve.argtypes = [i, i, _u64p, _vp, i, _u64p, _fp, i, _vp]
    for name in ("vk_rl_plan_create", "vk_rl_plan_shapes", "vk_rl_plan_device_bytes", "vk_rl_plan_launches",
                 "vk_rl_plan_destroy", "vk_rl_run", "vk_rl_run_device", "vk_rl_run_batch", "vk_rl_step",
                 "vk_rl_step_device", "vk_richardson_lucy", "vk_rl_step_psf", "vk_conv_plan_create",
                 "vk_conv_run", "vk_conv_run_device", "vk_fft_convolve"):
        getattr(L, name).restype = st
    L.vk_rl_plan_describe.argtypes = [_vp, ctypes.c_char_p, i]
    L.vk_rl_plan_describe.restype = st
    L.vk_rl_plan_profile.argtypes = [_vp, i]
    L.vk_rl_plan_profile_read.argtypes = [_vp, i, _dp, _u64p, _u64p, i]
    L.vk_rl_plan_profile.restype = st
    L.vk_rl_plan_profile_read.restype = st
    L.vk_volume_info_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(_VolumeInfo)]
    L.vk_volume_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(_VolumeInfo), _vp, ctypes.c_uint64]
    L.vk_volume_read_device.argtypes = [ctypes.c_char_p, ctypes.POINTER(_VolumeInfo), _vp, ctypes.c_uint64, _vp]
    L.vk_volume_write.argtypes = [ctypes.c_char_p, ctypes.POINTER(_VolumeInfo), _vp]
    L.vk_volume_write_device.argtypes = [ctypes.c_char_p, ctypes.POINTER(_VolumeInfo), _vp, _vp]
    L.vk_generate_blobs.argtypes = [i, ctypes.POINTER(_SynthSpec), _vp, _dp, _vp]
    L.vk_gaussian_psf.argtypes = [i, _u64p, _dp, i, _fp]
    for name in ("vk_volume_info_read", "vk_volume_read", "vk_volume_read_device", "vk_volume_write",
                 "vk_volume_write_device", "vk_generate_blobs", "vk_gaussian_psf"):
        getattr(L, name).restype = st
    L.vk_richardson_lucy_batch.argtypes = [i, i, _u64p, i, ctypes.POINTER(_vp), i, _u64p, _fp,
                                           ctypes.POINTER(_Rule), i, ctypes.POINTER(_vp), ctypes.POINTER(_Trace)]
    L.vk_richardson_lucy_batch.restype = st
    L.vk_rl_plan_otf_bytes.argtypes = [_vp, i, _u64p]
    L.vk_rl_plan_otf_bytes.restype = st
    L.vk_plan_cache_clear.argtypes = []
    L.vk_plan_cache_clear.restype = st
    L.vk_good_size.argtypes = [ctypes.c_uint64]
    L.vk_good_size.restype = ctypes.c_uint64
    L.vk_last_error.restype = ctypes.c_char_p
    L.vk_abi_version.restype = ctypes.c_int
    L.vk_debug_guard_check.argtypes = []
    L.vk_debug_guard_check.restype = ctypes.c_int
    _lib = L
    return L


def debug_guard_check() -> int:
    """With VK_RL_GUARD=1 set before the library is loaded: the number of
    device-buffer guard bands found overwritten so far (vk_debug_guard_check);
    -1 when guards are off."""
    return int(lib().vk_debug_guard_check())


def plan_cache_clear() -> None:
    """Frees the idle plans the one-shot calls (richardson_lucy, rl_step with a
    PSF, fft_convolve) keep for reuse (vk_plan_cache_clear)."""
    _check(lib().vk_plan_cache_clear())


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().vk_last_error().decode()
        raise _STATUS.get(rc, Error)(msg)


def _shape(s: Sequence[int]):
    return (ctypes.c_uint64 * max(len(s), 1))(*[int(v) for v in s])


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def good_size(n: int) -> int:
    """fftx::good_size (reference src/fft_plan.cpp:41-49)."""
    return int(lib().vk_good_size(int(n)))


# --- deconv types (reference: include/voxelkit/deconv.hpp:28-95) -----------
class StopMetric:
    si_psnr_vs_input = "si_psnr_vs_input"
    ssim_vs_prev = "ssim_vs_prev"
    frc_resolution = "frc_resolution"


_METRIC_ID = {StopMetric.si_psnr_vs_input: 0, StopMetric.ssim_vs_prev: 1, StopMetric.frc_resolution: 2}


def to_string(metric: str) -> str:
    return metric


@dataclass
class StoppingRule:
    metric: str = StopMetric.frc_resolution
    rel_tol: float = 1e-3
    patience: int = 3
    max_iters: int = 100

    def _c(self, spacing: Optional[float] = None) -> _Rule:
        """C struct; `spacing` is observed.spacing()->back() in the reference
        (used by frc_resolution), None = no spacing (1.0)."""
        return _Rule(_METRIC_ID[self.metric], float(self.rel_tol), int(self.patience), int(self.max_iters),
                     float(spacing) if spacing else 0.0)


@dataclass
class IterationRecord:
    iter: int
    metric_name: str
    value: float
    wall_time_s: float


@dataclass
class IterationTrace:
    records: List[IterationRecord] = field(default_factory=list)
    log_likelihood: List[float] = field(default_factory=list)
    fft_shape: tuple = ()
    stop_reason: str = "max_iters"

    def to_csv(self, out: Optional[io.TextIOBase] = None) -> str:
        """iter,metric,value,wall_time_s (reference src/deconv.cpp:85-96)."""
        lines = ["iter,metric,value,wall_time_s"]
        for r in self.records:
            v = ("inf" if r.value > 0 else "-inf") if math.isinf(r.value) else f"{r.value:.6g}"
            lines.append(f"{r.iter},{r.metric_name},{v},{r.wall_time_s:.6g}")
        s = "\n".join(lines) + "\n"
        if out is not None:
            out.write(s)
        return s


@dataclass
class RlResult:
    estimate: np.ndarray
    trace: IterationTrace


class _TraceBuf:
    def __init__(self, cap: int):
        self.m = np.zeros(cap)
        self.w = np.zeros(cap)
        self.ll = np.zeros(cap)
        self.c = _Trace(cap, self.m.ctypes.data_as(_dp), self.w.ctypes.data_as(_dp),
                        self.ll.ctypes.data_as(_dp), 0, 0)

    def trace(self, metric: str, rank: int) -> IterationTrace:
        n = self.c.iters_run
        recs = [IterationRecord(i + 1, metric, float(self.m[i]), float(self.w[i])) for i in range(n)]
        return IterationTrace(recs, [float(v) for v in self.ll[:n]],
                              tuple(int(self.c.fft_shape[i]) for i in range(rank)),
                              "converged" if self.c.stop_reason == 1 else "max_iters")


class _Plan:
    def __init__(self, shape, psf, pad: bool, device: int = 0, conv: int = 0):
        self._h = None
        k = _f32(psf)
        shape = tuple(int(s) for s in shape)
        h = _vp()
        if conv:
            _check(lib().vk_conv_plan_create(device, len(shape), _shape(shape), k.ndim, _shape(k.shape),
                                             k.ctypes.data_as(_fp), int(conv == 2), ctypes.byref(h)))
        else:
            _check(lib().vk_rl_plan_create(device, len(shape), _shape(shape), k.ndim, _shape(k.shape),
                                           k.ctypes.data_as(_fp), int(pad), ctypes.byref(h)))
        self._h = h
        self.device = device
        r = ctypes.c_int(0)
        im, dm, wm = (ctypes.c_uint64 * 3)(), (ctypes.c_uint64 * 3)(), (ctypes.c_uint64 * 3)()
        _check(lib().vk_rl_plan_shapes(h, ctypes.byref(r), im, dm, wm))
        self.rank = r.value
        self.image_shape_ = tuple(int(im[i]) for i in range(r.value))
        self.domain_shape = tuple(int(dm[i]) for i in range(r.value))
        self.fft_shape_ = tuple(int(wm[i]) for i in range(r.value))

    def launches(self) -> int:
        v = ctypes.c_uint64(0)
        _check(lib().vk_rl_plan_launches(self._h, ctypes.byref(v)))
        return int(v.value)

    def describe(self) -> str:
        """Execution plan chosen for this shape (kernel variant per axis, y/z strategy)."""
        buf = ctypes.create_string_buffer(512)
        _check(lib().vk_rl_plan_describe(self._h, buf, 512))
        return buf.value.decode()

    def profile(self, enable: bool = True) -> None:
        """CUDA-event timing of every launch, by kernel kind (vk_rl_plan_profile)."""
        _check(lib().vk_rl_plan_profile(self._h, int(bool(enable))))

    def profile_read(self, reset: bool = True) -> dict:
        """{kind: (total_ms, launches, algorithmic_bytes_per_launch)}."""
        n = len(KERNEL_KINDS)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_uint64 * n)()
        ab = (ctypes.c_uint64 * n)()
        _check(lib().vk_rl_plan_profile_read(self._h, n, ms, cnt, ab, int(bool(reset))))
        return {KERNEL_KINDS[i]: (float(ms[i]), int(cnt[i]), int(ab[i])) for i in range(n)}

    def otf_bytes(self) -> dict:
        """{kind: OTF bytes one launch reads} (not part of the algorithmic bytes)."""
        n = len(KERNEL_KINDS)
        ob = (ctypes.c_uint64 * n)()
        _check(lib().vk_rl_plan_otf_bytes(self._h, n, ob))
        return {KERNEL_KINDS[i]: int(ob[i]) for i in range(n)}

    def device_bytes(self) -> int:
        v = ctypes.c_uint64(0)
        _check(lib().vk_rl_plan_device_bytes(self._h, ctypes.byref(v)))
        return int(v.value)

    def close(self):
        if self._h is not None and _lib is not None:
            lib().vk_rl_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _checked_out(out: Optional[np.ndarray], shape) -> np.ndarray:
    """A caller-supplied output array must be a writable C-contiguous float32
    array of the plan's image shape: the C ABI writes prod(shape) floats."""
    if out is None:
        return np.empty(shape, np.float32)
    if not isinstance(out, np.ndarray) or out.dtype != np.float32 or tuple(out.shape) != tuple(shape) \
            or not out.flags.c_contiguous or not out.flags.writeable:
        raise ShapeMismatch(f"ShapeMismatch: out must be a writable C-contiguous float32 array of shape "
                            f"{list(shape)}")
    return out


def _check_image(a: np.ndarray, shape, what: str = "observed") -> None:
    if tuple(a.shape) != tuple(shape):
        raise ShapeMismatch(f"ShapeMismatch: {what} {list(a.shape)} vs plan {list(shape)}")


class RlTransforms(_Plan):
    """RlTransforms(image_shape, psf, threads) (reference src/deconv.cpp:98-176):
    PSF spectra for 'same' convolutions on `image_shape`, built once on the GPU.
    `threads` is accepted for signature parity; the device decides parallelism."""

    def __init__(self, image_shape, psf, threads: int = 1, device: int = 0):
        super().__init__(image_shape, psf, pad=False, device=device)

    def image_shape(self):
        return self.image_shape_

    def fft_shape(self):
        return self.fft_shape_


class RlPlan(_Plan):
    """Reusable richardson_lucy plan for one image shape + PSF (the padded
    domain, both OTFs and all work buffers stay resident on the GPU)."""

    def __init__(self, image_shape, psf, device: int = 0):
        super().__init__(image_shape, psf, pad=True, device=device)

    def run(self, observed, rule: StoppingRule = StoppingRule(), flat_init: bool = False,
            out: Optional[np.ndarray] = None) -> RlResult:
        obs = _f32(observed)
        _check_image(obs, self.image_shape_)
        est = _checked_out(out, self.image_shape_)
        tb = _TraceBuf(max(int(rule.max_iters), 1))
        _check(lib().vk_rl_run(self._h, obs.ctypes.data, est.ctypes.data, ctypes.byref(rule._c()),
                               int(bool(flat_init)), ctypes.byref(tb.c)))
        return RlResult(est, tb.trace(rule.metric, self.rank))

    def run_ptr(self, obs_ptr: int, est_ptr: int, rule: StoppingRule, flat_init: bool = False,
                trace: bool = True) -> Optional[IterationTrace]:
        """Host-pointer run (pinned or pageable) without numpy wrapping."""
        tb = _TraceBuf(max(int(rule.max_iters), 1)) if trace else None
        _check(lib().vk_rl_run(self._h, obs_ptr, est_ptr, ctypes.byref(rule._c()), int(bool(flat_init)),
                               ctypes.byref(tb.c) if tb else None))
        return tb.trace(rule.metric, self.rank) if tb else None

    def run_device(self, obs_ptr: int, est_ptr: int, rule: StoppingRule, flat_init: bool = False,
                   stream: int = 0, trace: bool = True) -> Optional[IterationTrace]:
        """Device-resident run: obs_ptr / est_ptr are CUDA device pointers on
        this plan's GPU (e.g. torch tensor .data_ptr()), stream a cudaStream_t."""
        tb = _TraceBuf(max(int(rule.max_iters), 1)) if trace else None
        _check(lib().vk_rl_run_device(self._h, obs_ptr, est_ptr, ctypes.byref(rule._c()), int(bool(flat_init)),
                                      ctypes.byref(tb.c) if tb else None, stream))
        return tb.trace(rule.metric, self.rank) if tb else None

    def run_batch_device(self, obs_ptrs: Sequence[int], est_ptrs: Sequence[int], rule: StoppingRule,
                         flat_init: bool = False, stream: int = 0, trace: bool = True):
        """Independent device-resident volumes, run concurrently on the plan's
        batch lanes (vk_rl_run_batch_device)."""
        n = len(obs_ptrs)
        tbs = [_TraceBuf(max(int(rule.max_iters), 1)) for _ in range(n)] if trace else None
        traces = (_Trace * max(n, 1))(*[t.c for t in tbs]) if trace else None
        ip = (_vp * max(n, 1))(*obs_ptrs)
        op = (_vp * max(n, 1))(*est_ptrs)
        _check(lib().vk_rl_run_batch_device(self._h, n, ip, op, ctypes.byref(rule._c()), int(bool(flat_init)),
                                            traces, stream))
        if not trace:
            return None
        out = []
        for i in range(n):
            tbs[i].c = traces[i]
            out.append(tbs[i].trace(rule.metric, self.rank))
        return out

    def lanes(self) -> int:
        v = ctypes.c_int(0)
        _check(lib().vk_rl_plan_lanes(self._h, ctypes.byref(v)))
        return int(v.value)

    def run_batch_ptr(self, obs_ptrs: Sequence[int], est_ptrs: Sequence[int], rule: StoppingRule,
                      flat_init: bool = False) -> None:
        """Host-pointer batch (vk_rl_run_batch): each lane copies its volume in
        (pinned host memory is DMA'd directly), runs it, and copies it out
        while the other lanes compute."""
        n = len(obs_ptrs)
        ip = (_vp * max(n, 1))(*obs_ptrs)
        op = (_vp * max(n, 1))(*est_ptrs)
        _check(lib().vk_rl_run_batch(self._h, n, ip, op, ctypes.byref(rule._c()), int(bool(flat_init)), None))

    def run_batch(self, observed: Sequence[np.ndarray], rule: StoppingRule = StoppingRule(),
                  flat_init: bool = False) -> List[RlResult]:
        obs = [_f32(o) for o in observed]
        for i, o in enumerate(obs):  # the C ABI copies prod(plan shape) floats per volume
            _check_image(o, self.image_shape_, f"observed[{i}]")
        outs = [np.empty_like(o) for o in obs]
        n = len(obs)
        tbs = [_TraceBuf(max(int(rule.max_iters), 1)) for _ in range(n)]
        traces = (_Trace * max(n, 1))(*[t.c for t in tbs])
        ip = (_vp * max(n, 1))(*[o.ctypes.data for o in obs])
        op = (_vp * max(n, 1))(*[o.ctypes.data for o in outs])
        _check(lib().vk_rl_run_batch(self._h, n, ip, op, ctypes.byref(rule._c()), int(bool(flat_init)), traces))
        res = []
        for i in range(n):
            tbs[i].c = traces[i]
            res.append(RlResult(outs[i], tbs[i].trace(rule.metric, self.rank)))
        return res


def richardson_lucy(observed, psf, rule: StoppingRule = StoppingRule(), flat_init: bool = False,
                    device: int = 0, spacing: Optional[Sequence[float]] = None) -> RlResult:
    """richardson_lucy (reference src/deconv.cpp:304-431) on the GPU.
    `spacing` mirrors NdImage::spacing() of the observed image (only its last
    entry is used, by the frc_resolution metric)."""
    obs = _f32(observed)
    k = _f32(psf)
    est = np.empty_like(obs)
    tb = _TraceBuf(max(int(rule.max_iters), 1))
    sp = float(spacing[-1]) if spacing is not None and len(spacing) else None
    _check(lib().vk_richardson_lucy(device, obs.ndim, _shape(obs.shape), obs.ctypes.data, k.ndim,
                                    _shape(k.shape), k.ctypes.data_as(_fp), ctypes.byref(rule._c(sp)),
                                    int(bool(flat_init)), est.ctypes.data, ctypes.byref(tb.c)))
    return RlResult(est, tb.trace(rule.metric, obs.ndim))


def richardson_lucy_batch(observed: Sequence[np.ndarray], psf, rule: StoppingRule = StoppingRule(),
                          flat_init: bool = False, device: int = 0) -> List[RlResult]:
    """richardson_lucy on each volume (one shape), through one cached plan and
    its batch lanes (vk_richardson_lucy_batch; reference semantics per volume,
    src/deconv.cpp:304-431)."""
    obs = [_f32(o) for o in observed]
    if not obs:
        return []
    for i, o in enumerate(obs):
        _check_image(o, obs[0].shape, f"observed[{i}]")
    k = _f32(psf)
    n = len(obs)
    outs = [np.empty_like(o) for o in obs]
    tbs = [_TraceBuf(max(int(rule.max_iters), 1)) for _ in range(n)]
    traces = (_Trace * n)(*[t.c for t in tbs])
    ip = (_vp * n)(*[o.ctypes.data for o in obs])
    op = (_vp * n)(*[o.ctypes.data for o in outs])
    _check(lib().vk_richardson_lucy_batch(device, obs[0].ndim, _shape(obs[0].shape), n, ip, k.ndim, _shape(k.shape),
                                          k.ctypes.data_as(_fp), ctypes.byref(rule._c()), int(bool(flat_init)), op,
                                          traces))
    res = []
    for i in range(n):
        tbs[i].c = traces[i]
        res.append(RlResult(outs[i], tbs[i].trace(rule.metric, obs[0].ndim)))
    return res


def _shape_str(s) -> str:
    return "[" + ",".join(str(int(v)) for v in s) + "]"


def rl_step(estimate, observed, transforms, device: int = 0) -> np.ndarray:
    """rl_step(estimate, observed, transforms | psf) (reference
    src/deconv.cpp:178-200): one multiplicative update, no padding."""
    e = _f32(estimate)
    o = _f32(observed)
    if e.shape != o.shape:  # require_same_shape (image.hpp:124-129)
        raise ShapeMismatch(f"ShapeMismatch: rl_step: {_shape_str(e.shape)} vs {_shape_str(o.shape)}")
    out = np.empty_like(e)
    if isinstance(transforms, RlTransforms):
        if e.shape != transforms.image_shape():
            raise ShapeMismatch("ShapeMismatch: rl_step: transforms were prepared for "
                                + _shape_str(transforms.image_shape()))
        _check(lib().vk_rl_step(transforms._h, e.ctypes.data, o.ctypes.data, out.ctypes.data))
        return out
    k = _f32(transforms)
    _check(lib().vk_rl_step_psf(device, e.ndim, _shape(e.shape), e.ctypes.data, o.ctypes.data, k.ndim,
                                _shape(k.shape), k.ctypes.data_as(_fp), out.ctypes.data))
    return out


class ConvPlan(_Plan):
    """filters::fft_convolve(img, kernel, circular) transforms for one image
    shape (reference src/filters.cpp:174-264): the kernel spectrum stays on the
    GPU; run() / run_device() convolve any image of that shape."""

    def __init__(self, image_shape, kernel, circular: bool = False, device: int = 0):
        super().__init__(image_shape, kernel, pad=False, device=device, conv=2 if circular else 1)
        self.circular = bool(circular)

    def run(self, image, out: Optional[np.ndarray] = None) -> np.ndarray:
        a = _f32(image)
        _check_image(a, self.image_shape_, "image")
        o = _checked_out(out, self.image_shape_)
        _check(lib().vk_conv_run(self._h, a.ctypes.data, o.ctypes.data))
        return o

    def run_device(self, img_ptr: int, out_ptr: int, stream: int = 0) -> None:
        _check(lib().vk_conv_run_device(self._h, img_ptr, out_ptr, stream))


def fft_convolve(image, kernel, circular: bool = False, device: int = 0) -> np.ndarray:
    """filters::fft_convolve (reference src/filters.cpp:174-264, registry op
    "fft_convolve" :316-323) on the GPU: linear mode returns the centred
    same-size result of the zero-padded convolution, circular mode the
    periodic convolution with the kernel centre at index 0."""
    a = _f32(image)
    k = _f32(kernel)
    out = np.empty_like(a)
    _check(lib().vk_fft_convolve(device, a.ndim, _shape(a.shape), a.ctypes.data, k.ndim, _shape(k.shape),
                                 k.ctypes.data_as(_fp), int(bool(circular)), out.ctypes.data))
    return out


# --- NDIV volumes and synthetic inputs (include/vk_io.h) ----------------------
_ELEM_DTYPE = {0: np.float32, 1: np.uint16, 2: np.uint32, 3: np.bool_}
_DTYPE_ELEM = {np.dtype(np.float32): 0, np.dtype(np.uint16): 1, np.dtype(np.uint32): 2, np.dtype(np.bool_): 3}


@dataclass
class Volume:
    """An NDIV volume: values (numpy, the file's element type) + spacing."""
    values: np.ndarray
    spacing: Optional[tuple] = None


def read_volume(path) -> Volume:
    """io::read_volume (reference src/io.cpp:83-158)."""
    info = _VolumeInfo()
    p = os.fsencode(path)
    _check(lib().vk_volume_info_read(p, ctypes.byref(info)))
    shape = tuple(int(info.shape[i]) for i in range(info.rank))
    out = np.empty(shape, _ELEM_DTYPE[info.elem])
    _check(lib().vk_volume_read(p, ctypes.byref(info), out.ctypes.data, out.nbytes))
    sp = tuple(float(info.spacing[i]) for i in range(info.rank)) if info.has_spacing else None
    return Volume(out, sp)


def _info_for(values: np.ndarray, spacing) -> _VolumeInfo:
    info = _VolumeInfo()
    if values.dtype not in _DTYPE_ELEM:
        raise Error(f"unsupported element type {values.dtype}")
    info.elem = _DTYPE_ELEM[values.dtype]
    info.rank = values.ndim
    if values.ndim > 4:
        raise HeaderMismatch(f"HeaderMismatch: unsupported rank {values.ndim}")
    for i, e in enumerate(values.shape):
        info.shape[i] = int(e)
    if spacing is not None:
        if len(spacing) != values.ndim:
            raise ShapeMismatch("ShapeMismatch: spacing needs one entry per axis")
        info.has_spacing = 1
        for i, v in enumerate(spacing):
            info.spacing[i] = float(v)
    return info


def write_volume(path, values, spacing=None) -> None:
    """io::write_volume (reference src/io.cpp:53-81); bytewise identical files."""
    a = np.ascontiguousarray(values)
    info = _info_for(a, spacing)
    _check(lib().vk_volume_write(os.fsencode(path), ctypes.byref(info), a.ctypes.data))


@dataclass
class VolumeInfo:
    shape: tuple
    dtype: type
    spacing: Optional[tuple] = None


def _py_info(info: _VolumeInfo) -> VolumeInfo:
    return VolumeInfo(tuple(int(info.shape[i]) for i in range(info.rank)), _ELEM_DTYPE[info.elem],
                      tuple(float(info.spacing[i]) for i in range(info.rank)) if info.has_spacing else None)


def volume_info(path) -> VolumeInfo:
    """Header of an NDIV file, fully validated (magic, JSON, payload length)."""
    info = _VolumeInfo()
    _check(lib().vk_volume_info_read(os.fsencode(path), ctypes.byref(info)))
    return _py_info(info)


def read_volume_device(path, dst_ptr: int, dst_bytes: int, stream: int = 0) -> VolumeInfo:
    """Stream the payload straight into device memory (pinned double
    buffering: the file read of one chunk overlaps the H2D of the other)."""
    info = _VolumeInfo()
    _check(lib().vk_volume_read_device(os.fsencode(path), ctypes.byref(info), dst_ptr, dst_bytes, stream))
    return _py_info(info)


def write_volume_device(path, src_ptr: int, shape, dtype=np.float32, spacing=None, stream: int = 0) -> None:
    """write_volume from device memory (D2H chunks overlap the file writes)."""
    info = _info_for(np.empty((0,) * len(tuple(shape)), dtype), spacing)
    for i, e in enumerate(shape):
        info.shape[i] = int(e)
    _check(lib().vk_volume_write_device(os.fsencode(path), ctypes.byref(info), src_ptr, stream))


@dataclass
class SynthSpec:
    """synth::SynthSpec (reference include/voxelkit/synth.hpp:27-39)."""
    shape: tuple = (32, 128, 128)
    n_objects: int = 20
    radius_min: float = 6.0
    radius_max: float = 10.0
    seed: int = 0
    noise_sigma: float = 0.05
    anisotropy: float = 1.0
    inplane_margin: float = 0.0

    def _c(self) -> _SynthSpec:
        if len(self.shape) != 3:
            raise Error("generate_blobs expects a 3D ZYX shape")
        return _SynthSpec((ctypes.c_uint64 * 3)(*[int(v) for v in self.shape]), int(self.n_objects),
                          float(self.radius_min), float(self.radius_max), int(self.seed),
                          float(self.noise_sigma), float(self.anisotropy), float(self.inplane_margin))


def generate_blobs_device(spec: SynthSpec, out_ptr: int, device: int = 0, stream: int = 0) -> tuple:
    """generate_blobs(spec).intensity into a device buffer; returns the spacing."""
    sp = (ctypes.c_double * 3)()
    c = spec._c()
    _check(lib().vk_generate_blobs(device, ctypes.byref(c), out_ptr, sp, stream))
    return tuple(sp)


def gaussian_psf(shape, sigmas) -> np.ndarray:
    """synth::gaussian_psf (reference src/synth.cpp:226-258)."""
    shape = tuple(int(s) for s in shape)
    sig = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, np.float64)))
    out = np.empty(shape, np.float32)
    _check(lib().vk_gaussian_psf(len(shape), _shape(shape), sig.ctypes.data_as(_dp), sig.size,
                                 out.ctypes.data_as(_fp)))
    return out


def exported_symbols() -> List[str]:
    """Function names declared in include/vk_rl.h (for the ABI tests)."""
    import re
    txt = ""
    for h in HEADER_PATHS:
        with open(h) as f:
            txt += f.read()
    return sorted(set(re.findall(r"^\s*(?:vk_status|uint64_t|const char\*|int)\s+(vk_\w+)\s*\(", txt, re.M)))


__all__ = [
    "Error", "ShapeMismatch", "NegativeInput", "UnnormalizedPsf", "DegenerateReference", "TooSmall",
    "OddExtent", "CudaError", "Unsupported", "KernelTooLarge", "ConvPlan", "fft_convolve", "StopMetric", "StoppingRule", "IterationRecord",
    "IterationTrace", "RlResult", "RlTransforms", "RlPlan", "richardson_lucy", "richardson_lucy_batch", "plan_cache_clear", "rl_step", "good_size",
    "to_string", "lib", "exported_symbols", "Volume", "VolumeInfo", "volume_info", "read_volume", "write_volume", "read_volume_device",
    "write_volume_device", "SynthSpec", "generate_blobs_device", "gaussian_psf", "BadMagic", "HeaderMismatch",
    "TruncatedPayload", "PlacementFailure", "EvenExtent",
]
