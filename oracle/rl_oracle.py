"""TEST INFRASTRUCTURE — numpy float64 restatement of the reference RL path.

This is the parity checker for the CUDA product path; only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import it, and
never as the thing measured or shipped.  Every function cites the reference
file:line it restates (paths relative to /root/reference/proj).  The FFT is
numpy's pocketfft in double precision, standing in for the reference's FFTW3
double r2c/c2r (src/fft_plan.cpp:84-97; FFTW unpinned and absent here) — the
two agree to ~1e-16 relative, invisible at f32 output.

Pinned against the reference itself: tests/test_oracle.py compares every
function here with oracle/_ref/libvkref.so (the reference sources compiled
unmodified by oracle/Makefile) and with the committed fixtures in
tests/golden/ produced by tests/golden/make_golden.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

K_DIV_EPSILON = 1e-12  # include/voxelkit/core_ops.hpp:26


class OracleError(Exception):
    """Mirrors the reference's typed errors: kind is the C++ class name."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}" if kind != "Error" else msg)
        self.kind = kind


def good_size(n: int) -> int:
    """Smallest 2^a 3^b 5^c >= n; good_size(<=1) = 1 (src/fft_plan.cpp:41-49)."""
    if n <= 1:
        return 1
    c = n
    while True:
        m = c
        for p in (2, 3, 5):
            while m % p == 0:
                m //= p
        if m == 1:
            return c
        c += 1


def kernel_center(extent: int) -> int:
    """(extent-1)/2 (src/deconv.cpp:40)."""
    return (extent - 1) // 2


def padded_domain(img_shape, psf_shape):
    """P = I + 2*floor(K/2), offset floor(K/2) (src/deconv.cpp:205-219)."""
    off = tuple(k // 2 for k in psf_shape)
    return tuple(i + 2 * o for i, o in zip(img_shape, off)), off


def replicate_pad(v: np.ndarray, off) -> np.ndarray:
    """Clamp-indexed gather into the padded domain (src/deconv.cpp:221-237)."""
    return np.pad(v.astype(np.float64), [(o, o) for o in off], mode="edge")


def crop_interior(v: np.ndarray, off, shape) -> np.ndarray:
    """P -> I window at floor(K/2), double -> f32 (src/deconv.cpp:239-252)."""
    sl = tuple(slice(o, o + s) for o, s in zip(off, shape))
    return v[sl].astype(np.float32)


class RlTransforms:
    """PSF spectra cached once per plan (src/deconv.cpp:98-131)."""

    def __init__(self, shape, psf: np.ndarray):
        psf = np.asarray(psf, dtype=np.float32)
        if psf.ndim != len(shape):
            raise OracleError("ShapeMismatch", "psf rank must match the image rank")
        self.image_shape = tuple(int(s) for s in shape)
        self.psf_shape = psf.shape
        # W = good_size(P + K - 1) per axis (src/deconv.cpp:114-116)
        self.fft_shape = tuple(good_size(s + k - 1) for s, k in zip(self.image_shape, psf.shape))
        k = psf.astype(np.float64)
        # corner_embed + r2c (src/deconv.cpp:126-130); std::reverse of the flat
        # buffer == flip about every axis.
        ax = tuple(range(k.ndim))
        self._axes = ax
        self.psf_fft = np.fft.rfftn(k, s=self.fft_shape, axes=ax)
        self.psf_flipped_fft = np.fft.rfftn(k[(slice(None, None, -1),) * k.ndim], s=self.fft_shape, axes=ax)
        self._crop = tuple(slice(kernel_center(kk), kernel_center(kk) + s)
                           for kk, s in zip(psf.shape, self.image_shape))

    def convolve(self, img: np.ndarray, flipped: bool) -> np.ndarray:
        """Linear 'same' convolution: corner_embed -> r2c -> x OTF -> c2r(1/N) ->
        centered_crop (src/deconv.cpp:135-147, src/fft_plan.cpp:84-97)."""
        spec = np.fft.rfftn(img, s=self.fft_shape, axes=self._axes)
        spec *= self.psf_flipped_fft if flipped else self.psf_fft
        full = np.fft.irfftn(spec, s=self.fft_shape, axes=self._axes)
        return full[self._crop]

    def step(self, estimate: np.ndarray, observed: np.ndarray) -> np.ndarray:
        """One multiplicative update (src/deconv.cpp:150-167)."""
        model = self.convolve(estimate, False)
        ratio = observed / np.maximum(model, K_DIV_EPSILON)
        correction = self.convolve(ratio, True)
        return np.maximum(estimate * correction, 0.0)


def rl_step(estimate, observed, psf) -> np.ndarray:
    """Registry form: unpadded transforms built per call, f32 in/out
    (src/deconv.cpp:178-200,437-449)."""
    e = np.asarray(estimate, np.float32)
    o = np.asarray(observed, np.float32)
    if e.shape != o.shape:
        raise OracleError("ShapeMismatch", f"rl_step: {list(e.shape)} vs {list(o.shape)}")
    t = RlTransforms(e.shape, psf)
    return t.step(e.astype(np.float64), o.astype(np.float64)).astype(np.float32)


def si_psnr(x: np.ndarray, ref: np.ndarray) -> float:
    """Scale-invariant PSNR (src/metrics.cpp:67-101), double accumulation."""
    a = np.asarray(x, np.float32).astype(np.float64).ravel()
    b = np.asarray(ref, np.float32).astype(np.float64).ravel()
    n = float(a.size)
    sx, sr, sxx, sxr, srr = a.sum(), b.sum(), (a * a).sum(), (a * b).sum(), (b * b).sum()
    var_r = srr / n - (sr / n) ** 2
    if var_r <= 0.0:
        raise OracleError("DegenerateReference", "si_psnr needs a non-constant reference")
    var_x = sxx / n - (sx / n) ** 2
    aa = (sxr / n - (sx / n) * (sr / n)) / var_x if var_x > 0.0 else 0.0
    bb = sr / n - aa * (sx / n)
    err = float(((aa * a + bb - b) ** 2).sum()) / n
    if err <= 0.0:
        return math.inf
    rng = float(b.max() - b.min())
    return 10.0 * math.log10(rng * rng / err)


def frc_curve(a: np.ndarray, b: np.ndarray, ring_width: float = 1.0):
    """metrics::frc (src/metrics.cpp:146-208): ring sums over the r2c
    half-spectra with weight 2 for conjugate-pair kx planes."""
    a = np.asarray(a, np.float32).astype(np.float64)
    b = np.asarray(b, np.float32).astype(np.float64)
    ax = tuple(range(a.ndim))
    sa, sb = np.fft.rfftn(a, axes=ax), np.fft.rfftn(b, axes=ax)
    shape = a.shape
    n_max = max(shape)
    bin_freq = ring_width / n_max
    n_bins = int(math.floor(0.5 / bin_freq)) + 1
    grids = np.meshgrid(*[np.arange(s) for s in sa.shape], indexing="ij")
    nu2 = np.zeros(sa.shape)
    for g, n in zip(grids, shape):
        nu2 += (np.minimum(g, n - g) / n) ** 2
    bins = np.rint(np.sqrt(nu2) / bin_freq)  # llround: ties away from zero
    half = np.sqrt(nu2) / bin_freq - np.floor(np.sqrt(nu2) / bin_freq) == 0.5
    bins = np.where(half, np.floor(np.sqrt(nu2) / bin_freq) + 1, bins).astype(np.int64)
    kx = grids[-1]
    selfc = (kx == 0) | ((shape[-1] % 2 == 0) & (kx == shape[-1] // 2))
    w = np.where(selfc, 1.0, 2.0)
    ok = bins < n_bins
    num = np.bincount(bins[ok], (w * (sa * np.conj(sb)).real)[ok], n_bins)
    da = np.bincount(bins[ok], (w * np.abs(sa) ** 2)[ok], n_bins)
    db = np.bincount(bins[ok], (w * np.abs(sb) ** 2)[ok], n_bins)
    den = np.sqrt(da * db)
    corr = np.where(den > 0, num / np.where(den > 0, den, 1), 0.0)
    return np.arange(n_bins) * bin_freq, corr


def frc_resolution(freq, corr, spacing: float, threshold: float = 1.0 / 7.0) -> float:
    """metrics::frc_resolution (src/metrics.cpp:210-239)."""
    for j in range(1, len(corr)):
        if corr[j] < threshold:
            if j == 1 or corr[j - 1] < threshold:
                nu = freq[j]
            else:
                nu = freq[j - 1] + (freq[j] - freq[j - 1]) * (corr[j - 1] - threshold) / (corr[j - 1] - corr[j])
            return math.inf if nu <= 0 else spacing / nu
    return math.inf


def single_image_frc(img: np.ndarray, spacing: float = 1.0) -> float:
    """even_view + metrics::single_image_frc (src/deconv.cpp:255-276,
    src/metrics.cpp:241-264)."""
    v = np.asarray(img, np.float32)
    v = v[tuple(slice(0, s - s % 2) for s in v.shape)]
    even = v[tuple(slice(0, None, 2) for _ in v.shape)]
    odd = v[tuple(slice(1, None, 2) for _ in v.shape)]
    f, c = frc_curve(even, odd)
    return frc_resolution(f, c, spacing * 2.0)


def gaussian_kernel_1d(sigma: float, truncate: float) -> np.ndarray:
    """filters.cpp:78-90: half = ceil(truncate*sigma) taps per side,
    exp(-0.5 (i/sigma)^2) normalised by their (sequential) sum."""
    half = int(math.ceil(truncate * sigma))
    w = [math.exp(-0.5 * (i / sigma) * (i / sigma)) for i in range(-half, half + 1)]
    tot = 0.0
    for v in w:
        tot += v
    return np.array([v / tot for v in w])


def mirror_index(i: np.ndarray, n: int) -> np.ndarray:
    """nd_utils.hpp:31-38 (reflect about the end samples, period 2(n-1))."""
    if n == 1:
        return np.zeros_like(i)
    period = 2 * (n - 1)
    m = np.mod(i, period)
    return np.where(m >= n, period - m, m)


def gaussian(img: np.ndarray, sigma: float = 1.5, truncate: float = 3.5) -> np.ndarray:
    """filters::gaussian (filters.cpp:92-140): one separable pass per axis,
    mirror boundary, double accumulation in tap order (each product and sum
    rounded separately, as the reference's scalar loop does), f32 result."""
    cur = np.asarray(img, np.float32).astype(np.float64)
    w = gaussian_kernel_1d(sigma, truncate)
    half = len(w) // 2
    for axis in range(cur.ndim):
        n = cur.shape[axis]
        idx = np.arange(n)
        acc = np.zeros_like(cur)
        for k in range(-half, half + 1):
            acc = acc + w[k + half] * np.take(cur, mirror_index(idx + k, n), axis=axis)
        cur = acc
    return cur.astype(np.float32)


def ssim(x: np.ndarray, ref: np.ndarray) -> float:
    """metrics::ssim (src/metrics.cpp:103-144) with the moments held alive
    (the reference reads them through dangling spans): five
    Gaussian-smoothed fields (sigma 1.5, truncate 3.5), c1 = (0.01 R)^2,
    c2 = (0.03 R)^2 with R = range of `ref`, mean of the SSIM map."""
    a = np.asarray(x, np.float32)
    b = np.asarray(ref, np.float32)
    if a.shape != b.shape:
        raise OracleError("ShapeMismatch", "ssim: shape mismatch")
    if any(e < 7 for e in a.shape):
        raise OracleError("TooSmall", "ssim needs every extent >= 7")
    rng = float(b.max()) - float(b.min())
    c1 = (0.01 * rng) * (0.01 * rng)
    c2 = (0.03 * rng) * (0.03 * rng)
    mx = gaussian(a).astype(np.float64)
    mr = gaussian(b).astype(np.float64)
    mxx = gaussian(a * a).astype(np.float64)  # f32 products (metrics.cpp:121-125)
    mrr = gaussian(b * b).astype(np.float64)
    mxr = gaussian(a * b).astype(np.float64)
    var_x = mxx - mx * mx
    var_r = mrr - mr * mr
    cov = mxr - mx * mr
    m = ((2 * mx * mr + c1) * (2 * cov + c2)) / ((mx * mx + mr * mr + c1) * (var_x + var_r + c2))
    return float(m.sum()) / float(a.size)


def relative_change(prev: float, cur: float) -> float:
    """src/deconv.cpp:296-300."""
    if math.isinf(prev) and math.isinf(cur) and prev == cur:
        return 0.0
    if math.isinf(prev) or math.isinf(cur):
        return math.inf
    return abs(cur - prev) / max(abs(prev), 1e-30)


@dataclass
class Trace:
    metric: list = field(default_factory=list)
    log_likelihood: list = field(default_factory=list)
    fft_shape: tuple = ()
    stop_reason: str = "max_iters"


def validate(observed, psf, rel_tol, patience, max_iters):
    """Validation order and messages of src/deconv.cpp:306-326."""
    if rel_tol <= 0 and not math.isinf(rel_tol):
        raise OracleError("Error", "rel_tol must be positive")
    if patience < 1:
        raise OracleError("Error", "patience must be >= 1")
    if max_iters < 1:
        raise OracleError("Error", "max_iters must be >= 1")
    obs = np.asarray(observed, np.float32)
    k = np.asarray(psf, np.float32)
    if obs.ndim != k.ndim:
        raise OracleError("ShapeMismatch", "psf rank must match the image rank")
    if (obs < 0).any():
        raise OracleError("NegativeInput", "observed image must be nonnegative")
    if (k < 0).any():
        raise OracleError("NegativeInput", "psf must be nonnegative")
    s = float(k.astype(np.float64).sum())
    if abs(s - 1.0) > 1e-3:
        raise OracleError("UnnormalizedPsf", "psf sums to %f" % s)
    return obs, k


def richardson_lucy(observed, psf, metric="si_psnr_vs_input", rel_tol=1e-3, patience=3,
                    max_iters=100, flat_init=False, iterates=None, spacing=1.0):
    """src/deconv.cpp:304-431 with all three stopping metrics (ssim_vs_prev
    compares with the previous iterate, the observed image at iteration 1,
    deconv.cpp:352,403,423).  If
    `iterates` is a list, the cropped f32 estimate after every iteration is
    appended to it."""
    obs, k = validate(observed, psf, rel_tol, patience, max_iters)
    if metric not in ("si_psnr_vs_input", "frc_resolution", "ssim_vs_prev"):
        raise NotImplementedError(metric)
    pshape, off = padded_domain(obs.shape, k.shape)
    t = RlTransforms(pshape, k)
    obs_p = replicate_pad(obs, off)
    est = np.full(pshape, obs_p.mean()) if flat_init else obs_p.copy()
    trace = Trace(fft_shape=t.fft_shape)
    inner = tuple(slice(o, o + s) for o, s in zip(off, obs.shape))
    ov = obs.astype(np.float64)
    fails, prev, have_prev = 0, 0.0, False
    previous = obs
    for it in range(1, max_iters + 1):
        model = t.convolve(est, False)
        m = np.maximum(model[inner], K_DIV_EPSILON)
        trace.log_likelihood.append(float((ov * np.log(m) - m).sum()))
        ratio = obs_p / np.maximum(model, K_DIV_EPSILON)
        est = np.maximum(est * t.convolve(ratio, True), 0.0)
        cur = crop_interior(est, off, obs.shape)
        if iterates is not None:
            iterates.append(cur)
        if metric == "si_psnr_vs_input":
            value = si_psnr(cur, obs)
        elif metric == "ssim_vs_prev":
            value = ssim(cur, previous)
        else:
            value = single_image_frc(cur, spacing)
        previous = cur
        trace.metric.append(value)
        if have_prev:
            fails = fails + 1 if relative_change(prev, value) < rel_tol else 0
            if fails >= patience:
                trace.stop_reason = "converged"
                break
        prev, have_prev = value, True
    return crop_interior(est, off, obs.shape), trace


def richardson_lucy_slabs(observed, psf, nslabs: int, iters: int, flat_init=False):
    """The §8(f4) slab decomposition restated on the CPU (test oracle): the
    padded domain is cut into `nslabs` z slabs; slab r owns P rows [z0, z1) and
    convolves over Q = [z0 - hb, z1 + ha) clipped to P with zeros outside,
    hb = Kz-1-cz, ha = cz, taking its halo rows from the neighbours (here: the
    global arrays).  Must equal richardson_lucy on the owned rows."""
    obs, k = validate(observed, psf, 1e-3, 1, iters)
    pshape, off = padded_domain(obs.shape, k.shape)
    obs_p = replicate_pad(obs, off)
    est = np.full(pshape, obs_p.mean()) if flat_init else obs_p.copy()
    Pz, Kz = pshape[0], k.shape[0]
    cz = kernel_center(Kz)
    hb, ha = Kz - 1 - cz, cz
    bounds = [(Pz * r // nslabs, Pz * (r + 1) // nslabs) for r in range(nslabs)]
    doms = [(max(0, z0 - hb), min(Pz, z1 + ha)) for z0, z1 in bounds]
    tfs = [RlTransforms((q1 - q0,) + pshape[1:], k) for q0, q1 in doms]
    for _ in range(iters):
        ratio = np.empty(pshape)
        for (z0, z1), (q0, q1), t in zip(bounds, doms, tfs):
            m = t.convolve(est[q0:q1], False)[z0 - q0:z1 - q0]
            ratio[z0:z1] = obs_p[z0:z1] / np.maximum(m, K_DIV_EPSILON)
        new = np.empty(pshape)
        for (z0, z1), (q0, q1), t in zip(bounds, doms, tfs):
            c = t.convolve(ratio[q0:q1], True)[z0 - q0:z1 - q0]
            new[z0:z1] = np.maximum(est[z0:z1] * c, 0.0)
        est = new
    return crop_interior(est, off, obs.shape)


def fft_convolve(img, kernel, circular=False) -> np.ndarray:
    """filters::fft_convolve (src/filters.cpp:175-264)."""
    a = np.asarray(img, np.float32).astype(np.float64)
    k = np.asarray(kernel, np.float32).astype(np.float64)
    if a.ndim != k.ndim:
        raise OracleError("ShapeMismatch", "fft_convolve: rank mismatch")
    if circular:
        if any(kk > s for kk, s in zip(k.shape, a.shape)):
            raise OracleError("KernelTooLarge", "circular convolution needs kernel <= image")
        W = a.shape
        kk = np.zeros(W)
        idx = np.indices(k.shape).reshape(k.ndim, -1)
        dst = tuple((idx[ax] - kernel_center(k.shape[ax])) % W[ax] for ax in range(k.ndim))
        kk[dst] = k.ravel()
        ax = tuple(range(a.ndim))
        out = np.fft.irfftn(np.fft.rfftn(a, axes=ax) * np.fft.rfftn(kk, axes=ax), s=W, axes=ax)
        return out.astype(np.float32)
    W = tuple(good_size(s + kk - 1) for s, kk in zip(a.shape, k.shape))
    ax = tuple(range(a.ndim))
    full = np.fft.irfftn(np.fft.rfftn(a, s=W, axes=ax) * np.fft.rfftn(k, s=W, axes=ax), s=W, axes=ax)
    sl = tuple(slice(kernel_center(kk), kernel_center(kk) + s) for kk, s in zip(k.shape, a.shape))
    return full[sl].astype(np.float32)


def gaussian_psf(shape, sigmas) -> np.ndarray:
    """Centered separable Gaussian, unit sum in double then f32
    (src/synth.cpp:226-258)."""
    sig = list(np.atleast_1d(sigmas).astype(float))
    if len(sig) == 1 and len(shape) > 1:
        sig = sig * len(shape)
    v = np.ones((), np.float64)
    for ext, s in zip(shape, sig):
        d = np.arange(ext, dtype=np.float64) - ext // 2
        g = (d == 0).astype(np.float64) if s <= 0 else np.exp(-0.5 * (d / s) * (d / s))
        v = np.multiply.outer(v, g)
    return (v / v.sum()).astype(np.float32)


def widefield_psf(k: int = 31) -> np.ndarray:
    """The C2 'widefield' PSF of SURVEY.md §8(d): per-plane 2D Gaussians with
    sigma(dz) = 1.5*sqrt(1+((dz*(1+0.15*sgn dz))/4)^2), each plane unit-sum,
    weighted exp(-|dz|/8), normalised in double then cast to f32.  Non-separable
    and axially asymmetric, so it exercises the flipped-PSF path."""
    h = k // 2
    d = np.arange(-h, h + 1, dtype=np.float64)
    out = np.zeros((k, k, k))
    for i, dz in enumerate(d):
        s = 1.5 * math.sqrt(1.0 + ((dz * (1.0 + 0.15 * np.sign(dz))) / 4.0) ** 2)
        g = np.exp(-0.5 * (d / s) ** 2)
        plane = np.multiply.outer(g, g)
        out[i] = plane / plane.sum() * math.exp(-abs(dz) / 8.0)
    return (out / out.sum()).astype(np.float32)
