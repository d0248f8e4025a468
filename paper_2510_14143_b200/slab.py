"""Single-volume slab decomposition of richardson_lucy.

The padded domain P of one 3D volume is cut into z slabs, one slab plan per
GPU (or several on one GPU), through the vk_rl_slab_* C ABI (include/vk_rl.h).
Each slab computes on its owned P rows plus the correlations' reach (Kz-1-cz
rows below, cz above); after every x pass the halo rows of its x-spectrum are
refreshed with the neighbours' owned rows.  With one process per GPU that is a
pair of torch.distributed send/recv per neighbour and pass (NCCL over NVLink);
in one process it is a peer/device copy.  Per-slab sums (observed statistics,
log-likelihood and si_psnr sums) are added up by the caller (all-reduce), and
the stopping rule (reference src/deconv.cpp:296-300, 400-423) runs here.

Slabs help when a volume does not fit one GPU or to cut its latency; the
batch configs use independent volumes per GPU instead (dist.py).  Only the
si_psnr_vs_input metric is supported in slab mode.
"""
from __future__ import annotations

import ctypes
import math
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import (DegenerateReference, Error, IterationRecord, IterationTrace, NegativeInput, RlResult, StopMetric,
               StoppingRule, Unsupported, UnnormalizedPsf, _check, _f32, _fp, _shape, _vp, lib)


class _SlabInfo(ctypes.Structure):
    _fields_ = [("own_begin", ctypes.c_int), ("own_end", ctypes.c_int), ("domain_begin", ctypes.c_int),
                ("domain_end", ctypes.c_int), ("image_begin", ctypes.c_int), ("image_end", ctypes.c_int),
                ("halo_below", ctypes.c_int), ("halo_above", ctypes.c_int), ("spectrum", ctypes.c_void_p),
                ("kx_planes", ctypes.c_uint64), ("rows", ctypes.c_uint64), ("row_elems", ctypes.c_uint64)]


_bound = False


def _bind() -> ctypes.CDLL:
    global _bound
    L = lib()
    if not _bound:
        i, d = ctypes.c_int, ctypes.POINTER(ctypes.c_double)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.vk_rl_slab_plan_create.argtypes = [i, u64p, u64p, ctypes.POINTER(ctypes.c_float), i, i,
                                             ctypes.POINTER(_vp), ctypes.POINTER(_SlabInfo)]
        L.vk_rl_slab_begin.argtypes = [_vp, _vp, d, _vp]
        L.vk_rl_slab_start.argtypes = [_vp, i, i, ctypes.c_double, _vp]
        L.vk_rl_slab_forward.argtypes = [_vp, _vp, i, _vp]
        L.vk_rl_slab_backward.argtypes = [_vp, _vp, i, _vp, _vp]
        L.vk_rl_slab_crop.argtypes = [_vp, _vp, _vp]
        L.vk_rl_slab_sums.argtypes = [_vp, i, d, _vp]
        L.vk_rl_slab_pack.argtypes = [_vp, i, i, _vp, _vp]
        L.vk_rl_slab_unpack.argtypes = [_vp, i, i, _vp, _vp]
        L.vk_rl_slab_copy_rows.argtypes = [_vp, i, _vp, i, i, _vp]
        for n in ("vk_rl_slab_plan_create", "vk_rl_slab_begin", "vk_rl_slab_start", "vk_rl_slab_forward",
                  "vk_rl_slab_backward", "vk_rl_slab_crop", "vk_rl_slab_sums", "vk_rl_slab_pack",
                  "vk_rl_slab_unpack", "vk_rl_slab_copy_rows"):
            getattr(L, n).restype = ctypes.c_int
        _bound = True
    return L


class SlabPlan:
    """One slab of a volume (vk_rl_slab_plan_create)."""

    def __init__(self, shape, psf, nslabs: int, slab: int, device: int = 0):
        L = _bind()
        k = _f32(psf)
        shape = tuple(int(s) for s in shape)
        if len(shape) != 3 or k.ndim != 3:
            raise Unsupported("slab decomposition needs a 3D volume and PSF")
        self._h = None
        h, info = _vp(), _SlabInfo()
        _check(L.vk_rl_slab_plan_create(device, _shape(shape), _shape(k.shape), k.ctypes.data_as(_fp), nslabs,
                                        slab, ctypes.byref(h), ctypes.byref(info)))
        self._h = h
        self.device, self.shape, self.nslabs, self.slab = device, shape, nslabs, slab
        self.own = (info.own_begin, info.own_end)
        self.domain = (info.domain_begin, info.domain_end)
        self.image = (info.image_begin, info.image_end)
        self.halo_below, self.halo_above = info.halo_below, info.halo_above
        self.rows, self.kx_planes, self.row_elems = int(info.rows), int(info.kx_planes), int(info.row_elems)
        self.own_local = (self.own[0] - self.domain[0], self.own[1] - self.domain[0])
        self.image_voxels = (self.image[1] - self.image[0]) * shape[1] * shape[2]

    def row_bytes(self, n: int) -> int:
        return self.kx_planes * n * self.row_elems * 8

    def begin(self, obs_ptr: int, stream: int) -> np.ndarray:
        st = np.zeros(8)
        _check(lib().vk_rl_slab_begin(self._h, obs_ptr, st.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), stream))
        return st

    def start(self, iters: int, flat_init: bool, mean: float, stream: int) -> None:
        _check(lib().vk_rl_slab_start(self._h, iters, int(bool(flat_init)), float(mean), stream))

    def forward(self, obs_ptr: int, it: int, stream: int) -> None:
        _check(lib().vk_rl_slab_forward(self._h, obs_ptr, it, stream))

    def backward(self, obs_ptr: int, it: int, out_ptr: Optional[int], stream: int) -> None:
        _check(lib().vk_rl_slab_backward(self._h, obs_ptr, it, out_ptr, stream))

    def crop(self, out_ptr: int, stream: int) -> None:
        _check(lib().vk_rl_slab_crop(self._h, out_ptr, stream))

    def sums(self, iters: int, stream: int) -> np.ndarray:
        acc = np.zeros((max(iters, 1), 4))
        _check(lib().vk_rl_slab_sums(self._h, iters, acc.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), stream))
        return acc[:iters]

    def pack(self, row: int, n: int, buf_ptr: int, stream: int) -> None:
        _check(lib().vk_rl_slab_pack(self._h, row, n, buf_ptr, stream))

    def unpack(self, row: int, n: int, buf_ptr: int, stream: int) -> None:
        _check(lib().vk_rl_slab_unpack(self._h, row, n, buf_ptr, stream))

    def close(self):
        if self._h is not None:
            lib().vk_rl_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def copy_halos(plans: Sequence[SlabPlan], stream: int) -> None:
    """Refresh every halo of adjacent in-process slabs (peer / device copies)."""
    L = _bind()
    for lo, hi in zip(plans[:-1], plans[1:]):
        # the upper slab's halo_below <- the lower slab's last owned rows
        n = hi.halo_below
        _check(L.vk_rl_slab_copy_rows(lo._h, lo.own_local[1] - n, hi._h, 0, n, stream))
        # the lower slab's halo_above <- the upper slab's first owned rows
        n = lo.halo_above
        _check(L.vk_rl_slab_copy_rows(hi._h, hi.own_local[0], lo._h, lo.rows - n, n, stream))


def halo_rows(kz: int):
    """(rows below, rows above) a slab reaches: Kz-1-cz and cz (deconv.cpp:40)."""
    ha = (kz - 1) // 2
    return kz - 1 - ha, ha


class DistHalo:
    """Halo exchange of this rank's slab with ranks r-1 / r+1 over
    torch.distributed: pack the owned boundary rows of S_A, batched
    isend/irecv with both neighbours (NCCL over NVLink on GPU buffers), unpack
    into the halo rows.  `kz` is the PSF's z extent."""

    def __init__(self, plan: SlabPlan, dist, torch, kz: int, device=None):
        self.p, self.dist, self.torch = plan, dist, torch
        self.dev = torch.device("cuda", plan.device) if device is None else torch.device(device)
        r, R = plan.slab, plan.nslabs
        self.lower, self.upper = (r - 1 if r > 0 else None), (r + 1 if r + 1 < R else None)
        hb, ha = halo_rows(kz)
        # the lower neighbour's halo_above is `ha` rows, the upper's halo_below `hb`
        self.n_to_lower = ha if self.lower is not None else 0
        self.n_to_upper = hb if self.upper is not None else 0
        mk = lambda n: torch.empty(max(plan.row_bytes(n) // 4, 1), dtype=torch.float32, device=self.dev)  # noqa: E731
        self.send_lo, self.send_hi = mk(self.n_to_lower), mk(self.n_to_upper)
        self.recv_lo, self.recv_hi = mk(plan.halo_below), mk(plan.halo_above)

    def _sync(self):
        if self.dev.type == "cuda":
            self.torch.cuda.synchronize(self.dev)

    def exchange(self, stream: int) -> None:
        p, dist = self.p, self.dist
        if self.lower is not None:
            p.pack(p.own_local[0], self.n_to_lower, self.send_lo.data_ptr(), stream)
        if self.upper is not None:
            p.pack(p.own_local[1] - self.n_to_upper, self.n_to_upper, self.send_hi.data_ptr(), stream)
        self._sync()
        ops = []
        if self.lower is not None:
            ops += [dist.P2POp(dist.isend, self.send_lo, self.lower), dist.P2POp(dist.irecv, self.recv_lo, self.lower)]
        if self.upper is not None:
            ops += [dist.P2POp(dist.isend, self.send_hi, self.upper), dist.P2POp(dist.irecv, self.recv_hi, self.upper)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        self._sync()
        if self.lower is not None:
            p.unpack(0, p.halo_below, self.recv_lo.data_ptr(), stream)
        if self.upper is not None:
            p.unpack(p.rows - p.halo_above, p.halo_above, self.recv_hi.data_ptr(), stream)


def dist_allreduce(dist, torch, device):
    """allreduce(array, op) for run_slabs over the default process group."""
    ops = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}

    def f(a: np.ndarray, op: str) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(device)
        dist.all_reduce(t, op=ops[op])
        return t.cpu().numpy()
    return f


# ---- the driver ------------------------------------------------------------------
def _relative_change(prev: float, cur: float) -> float:  # deconv.cpp:296-300
    if math.isinf(prev) and math.isinf(cur) and prev == cur:
        return 0.0
    if math.isinf(prev) or math.isinf(cur):
        return math.inf
    return abs(cur - prev) / max(abs(prev), 1e-30)


def _si_psnr(n, sr, srr, rng, sx, sxx, sxr) -> float:  # metrics.cpp:67-101 from sums
    var_r = srr / n - (sr / n) ** 2
    if var_r <= 0.0:
        raise DegenerateReference("DegenerateReference: si_psnr needs a non-constant reference")
    var_x = sxx / n - (sx / n) ** 2
    cov = sxr / n - (sx / n) * (sr / n)
    a = cov / var_x if var_x > 0.0 else 0.0
    err = var_r - a * cov
    if err <= 0.0:
        return math.inf
    return 10.0 * math.log10(rng * rng / err)


def _check_rule(rule: StoppingRule) -> None:  # deconv.cpp:306-311
    if rule.rel_tol <= 0 and not math.isinf(rule.rel_tol):
        raise Error("rel_tol must be positive")
    if rule.patience < 1:
        raise Error("patience must be >= 1")
    if rule.max_iters < 1:
        raise Error("max_iters must be >= 1")
    if rule.metric != StopMetric.si_psnr_vs_input:
        raise Unsupported("slab decomposition supports the si_psnr_vs_input metric only")


def _check_psf(psf: np.ndarray) -> None:  # deconv.cpp:319-326
    k = np.asarray(psf, np.float32)
    if (k < 0).any():
        raise NegativeInput("NegativeInput: psf must be nonnegative")
    s = float(k.astype(np.float64).sum())
    if abs(s - 1.0) > 1e-3:
        raise UnnormalizedPsf("UnnormalizedPsf: psf sums to %f" % s)


def _rule_stops(values: Sequence[float], rule: StoppingRule) -> bool:
    """Replays the stopping rule over metric values 1..n (deconv.cpp:409-423)."""
    fails, have_prev, prev = 0, False, 0.0
    for v in values:
        if have_prev:
            fails = fails + 1 if _relative_change(prev, v) < rule.rel_tol else 0
            if fails >= rule.patience:
                return True
        prev, have_prev = v, True
    return False


def run_slabs(plans: Sequence[SlabPlan], obs_ptrs: Sequence[int], out_ptrs: Sequence[int], psf,
              rule: StoppingRule, flat_init: bool, exchange: Callable[[int], None],
              allreduce: Callable[[np.ndarray, str], np.ndarray], stream: int = 0) -> IterationTrace:
    """richardson_lucy (reference src/deconv.cpp:304-431) over the slabs this
    process holds.  obs_ptrs / out_ptrs: device pointers to each slab's own
    image rows.  exchange(stream) refreshes every halo; allreduce(array, op)
    reduces an array over all slabs of the volume in other processes ("sum",
    "min" or "max"; identity when every slab is local)."""
    _check_rule(rule)
    st = [p.begin(o, stream) for p, o in zip(plans, obs_ptrs)]
    sums = allreduce(np.array([sum(x[k] for x in st) for k in (0, 1, 4, 5, 6, 7)]), "sum")
    vmin = float(allreduce(np.array([min(x[2] for x in st)]), "min")[0])
    vmax = float(allreduce(np.array([max(x[3] for x in st)]), "max")[0])
    sr, srr, sump, neg, n_img, n_pad = sums
    if neg > 0:
        raise NegativeInput("NegativeInput: observed image must be nonnegative")
    _check_psf(psf)
    rng = vmax - vmin
    _si_psnr(n_img, sr, srr, rng, 0.0, 0.0, 0.0)  # DegenerateReference before any estimate
    iters = int(rule.max_iters)
    mean = sump / n_pad
    for p in plans:
        p.start(iters, flat_init, mean, stream)
    exchange(stream)
    may_stop = rule.patience + 1 <= iters
    values: List[float] = []
    run, stopped = 0, False
    for it in range(1, iters + 1):
        for p, o in zip(plans, obs_ptrs):
            p.forward(o, it, stream)
        exchange(stream)
        last = it == iters
        for p, o, out in zip(plans, obs_ptrs, out_ptrs):
            p.backward(o, it, out if last else None, stream)
        run = it
        if may_stop and it >= rule.patience + 1 and not last:
            acc = allreduce(sum(p.sums(it, stream) for p in plans), "sum")
            values = [_si_psnr(n_img, sr, srr, rng, a[1], a[2], a[3]) for a in acc]
            stopped = _rule_stops(values, rule)
            if stopped:
                for p, out in zip(plans, out_ptrs):
                    p.crop(out, stream)
                break
        if not last:
            exchange(stream)
    acc = allreduce(sum(p.sums(run, stream) for p in plans), "sum")
    recs = [IterationRecord(i + 1, StopMetric.si_psnr_vs_input, _si_psnr(n_img, sr, srr, rng, a[1], a[2], a[3]), 0.0)
            for i, a in enumerate(acc)]
    # the reference checks the rule on the last iteration too (deconv.cpp:409-423):
    # a run that converges exactly at max_iters reports "converged"
    if not stopped:
        stopped = _rule_stops([r.value for r in recs], rule)
    return IterationTrace(recs, [float(a[0]) for a in acc], (), "converged" if stopped else "max_iters")


def richardson_lucy_slabs(observed, psf, rule: StoppingRule, flat_init: bool = False, nslabs: int = 2,
                          device: int = 0) -> RlResult:
    """One volume, `nslabs` slab plans in this process on one GPU (the
    single-process form of the decomposition; the multi-GPU form runs one
    SlabPlan per rank with DistHalo and an NCCL all-reduce)."""
    import torch

    obs = _f32(observed)
    k = _f32(psf)
    plans = [SlabPlan(obs.shape, k, nslabs, r, device) for r in range(nslabs)]
    d_obs = torch.from_numpy(obs).to(torch.device("cuda", device))
    d_out = torch.empty_like(d_obs)
    ptr = lambda t, r: t.data_ptr() + r * obs.shape[1] * obs.shape[2] * 4  # noqa: E731
    s = torch.cuda.current_stream(device).cuda_stream
    tr = run_slabs(plans, [ptr(d_obs, p.image[0]) for p in plans], [ptr(d_out, p.image[0]) for p in plans], k, rule,
                   flat_init, lambda st: copy_halos(plans, st), lambda a, op: a, s)
    torch.cuda.synchronize(device)
    for p in plans:
        p.close()
    return RlResult(d_out.cpu().numpy(), tr)
