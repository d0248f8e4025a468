"""Synthetic inputs shaped like the benchmark configs.

Values do not affect throughput; parity only needs both sides to see the
same input.  A numpy soft-disk/ellipsoid phantom is used so nothing here
depends on the reference being present on the GPU box.
"""
from __future__ import annotations

import numpy as np


def blobs(shape, n, rmin, rmax, seed, noise=0.05):
    """Soft-edged ellipsoids (2-voxel cosine taper, like src/synth.cpp:181-186)
    plus Gaussian noise; any rank 1..3."""
    rng = np.random.default_rng(seed)
    shape = tuple(int(s) for s in shape)
    img = np.zeros(shape, np.float64)
    for _ in range(n):
        r = rng.uniform(rmin, rmax)
        c = [rng.uniform(min(r + 3, s / 2), max(s - 1 - r - 3, s / 2)) for s in shape]
        lo = [max(0, int(cc - r - 2)) for cc in c]
        hi = [min(s, int(cc + r + 3)) for cc, s in zip(c, shape)]
        box = tuple(slice(a, b) for a, b in zip(lo, hi))
        grids = np.meshgrid(*[np.arange(a, b, dtype=np.float64) for a, b in zip(lo, hi)], indexing="ij")
        rho = np.sqrt(sum(((g - cc) / r) ** 2 for g, cc in zip(grids, c)))
        hb = 1.0 / r
        prof = np.where(rho <= 1 - hb, 1.0,
                        np.where(rho >= 1 + hb, 0.0, 0.5 * (1 + np.cos(np.pi * (rho - (1 - hb)) / (2 * hb)))))
        img[box] = np.maximum(img[box], prof)
    img += noise * rng.standard_normal(shape)
    return img.astype(np.float32)


def blurred(truth, psf):
    """observed = max(fft_convolve(truth, psf), 0) as the reference CLI builds it
    (tools/voxelkit_main.cpp:417-425), using the numpy oracle's convolution."""
    from oracle import rl_oracle

    return np.maximum(rl_oracle.fft_convolve(truth, psf), 0).astype(np.float32)
