#!/usr/bin/env python
"""Small runs of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck): fast x/y/z passes with TMA / bulk copies /
mbarriers / PDL, the generic Stockham kernels, FRC and SSIM metrics, batch
lanes, the circular fft_convolve extension.  Sizes are chosen so the
compile-time FFT lengths the configs use (96, 192, 288, 576) are exercised.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [small|full]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2510_14143_b200 as vk  # noqa: E402
from oracle import rl_oracle as O  # noqa: E402


def gauss(shape, s):
    return O.gaussian_psf(shape, s)


def run(obs, psf, metric="si_psnr_vs_input", iters=2, flat=False):
    r = vk.richardson_lucy(obs, psf, vk.StoppingRule(metric, 1e-300, iters, iters), flat)
    assert np.isfinite(r.estimate).all()
    print(metric, obs.shape, psf.shape, r.trace.fft_shape, [round(x.value, 4) for x in r.trace.records], flush=True)


def main(mode):
    rng = np.random.default_rng(0)
    vol = lambda s: (rng.random(s) + 0.1).astype(np.float32)  # noqa: E731
    # 96^3 grid: fast x (TMA-less 96), y bulk, z TMA at 96
    run(vol((88, 88, 88)), gauss((5, 5, 5), 1.0))
    # generic Stockham path (180 is not a compile-time length), flat_init
    run(vol((20, 60, 70)), gauss((5, 7, 9), 1.2), flat=True)
    # 2D: 288 grid (TMA x pass), y convolution, factored OTF
    run(vol((258, 258)), gauss((31, 31), 3.75))
    # metrics on device
    run(vol((24, 40, 48)), gauss((5, 5, 5), 1.0), "frc_resolution", 3)
    run(vol((24, 40, 48)), gauss((5, 5, 5), 1.0), "ssim_vs_prev", 3)
    # non-separable PSF (full OTF read through the TMA OTF tile), 192 z / 576 x,y at full mode
    if mode == "full":
        run(vol((132, 516, 516)), O.widefield_psf(31), iters=1)
    else:
        run(vol((40, 90, 100)), O.widefield_psf(9), iters=2)
    # batch lanes (host threads + streams)
    k = gauss((5, 5), 1.0)
    res = vk.richardson_lucy_batch([vol((100, 120)) for _ in range(4)], k,
                                   vk.StoppingRule("si_psnr_vs_input", 1e-300, 2, 2))
    print("batch", len(res), flush=True)
    # fft_convolve: linear, circular 5-smooth, circular any extent
    a = vol((30, 40, 50))
    for circ, shape in ((False, (30, 40, 50)), (True, (30, 40, 50)), (True, (7, 11, 13))):
        x = vol(shape)
        y = vk.fft_convolve(x, gauss((3, 3, 3), 1.0), circular=circ)
        assert np.isfinite(y).all()
    print("fft_convolve ok", a.shape, flush=True)
    # the benchmarked paths: kx-chunked y/z convolution at the C2 grid
    # (576 x / y, 192 z, half OTF), the C4 grid (1080 x TMA pass), a 2160-point
    # 2D field, device-side stopping (CUDA graph), rl_step
    os.environ["VK_RL_KXCHUNK"] = "2"
    run(vol((128, 512, 60)), O.widefield_psf(31), iters=2)
    run(vol((100, 1000, 20)), gauss((21, 21, 21), 2.5), iters=2)
    del os.environ["VK_RL_KXCHUNK"]
    if mode == "full":
        run(vol((2048, 2048)), gauss((31, 31), 3.75), iters=2)
    r = vk.richardson_lucy(vol((24, 48, 40)), gauss((7, 7, 7), 1.2), vk.StoppingRule("si_psnr_vs_input", 1e-2, 2, 12))
    print("graph stop", len(r.trace.records), r.trace.stop_reason, flush=True)
    e, o = vol((20, 30, 40)), vol((20, 30, 40))
    assert np.isfinite(vk.rl_step(e, o, gauss((5, 5, 5), 1.0))).all()
    vk.plan_cache_clear()
    print("GUARD_VIOLATIONS", vk.debug_guard_check(), flush=True)
    print("SANITIZE_CASES_DONE")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
