"""Generate the committed golden fixtures from the reference itself.

Runs the reference's own richardson_lucy / rl_step / fft_convolve (compiled
unmodified from /root/reference by oracle/Makefile into oracle/_ref/libvkref.so)
on small seeded inputs and stores inputs + outputs in tests/golden/*.npz.
Re-run with:  make -C oracle && python tests/golden/make_golden.py
The fixtures travel to the GPU box; the reference tree does not.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FIXED = dict(rel_tol=1e-300)  # fixed iteration count: patience = max_iters


def blur_observed(truth, psf):
    # observed = vmax(fft_convolve(truth, psf), 0) as the reference CLI builds it
    # (tools/voxelkit_main.cpp:417-425)
    return np.maximum(ref.fft_convolve(truth, psf), 0).astype(np.float32)


def rl_case(name, observed, psf, iters, flat_init=False, metric="si_psnr_vs_input", **rule):
    kw = dict(FIXED, patience=iters, max_iters=iters)
    kw.update(rule)
    r1 = ref.richardson_lucy(observed, psf, metric=metric, flat_init=flat_init,
                             **dict(kw, max_iters=1, patience=1))
    rn = ref.richardson_lucy(observed, psf, metric=metric, flat_init=flat_init, **kw)
    np.savez_compressed(
        os.path.join(OUT, f"rl_{name}.npz"), observed=observed, psf=psf,
        estimate_1=r1.estimate, estimate_n=rn.estimate, metric=rn.metric,
        loglik=rn.loglik, iters_run=rn.iters_run, stop_reason=rn.stop_reason,
        fft_shape=np.array(rn.fft_shape), flat_init=flat_init, metric_name=metric,
        rel_tol=kw["rel_tol"], patience=kw["patience"], max_iters=kw["max_iters"])
    print(name, observed.shape, psf.shape, rn.fft_shape, rn.iters_run, rn.stop_reason)


def main():
    rng = np.random.default_rng(20261018)

    # 3D blob phantom, odd Gaussian PSF (C1 regime at reduced size)
    truth = ref.generate_blobs((20, 48, 48), n_objects=4, radius_min=3, radius_max=5, seed=7,
                               noise_sigma=0.05)
    psf = ref.gaussian_psf((7, 7, 7), [1.0])
    rl_case("blobs3d", blur_observed(truth, psf), psf, 6)
    rl_case("blobs3d_flat", blur_observed(truth, psf), psf, 4, flat_init=True)

    # even PSF extents (one-sample-shifted correlation)
    obs = (rng.random((6, 20, 22)) * 2).astype(np.float32)
    k = rng.random((4, 6, 6))
    rl_case("even3d", obs, (k / k.sum()).astype(np.float32), 4)

    # odd FFT length (W = 45 on the last axis)
    obs = (rng.random((5, 9, 33)) + 0.1).astype(np.float32)
    k = rng.random((3, 3, 5))
    rl_case("oddw", obs, (k / k.sum()).astype(np.float32), 3)

    # non-separable, axially asymmetric PSF (flip path)
    k = rng.random((5, 5, 5)) ** 3
    obs = (rng.random((10, 18, 20)) * 5).astype(np.float32)
    rl_case("asym3d", obs, (k / k.sum()).astype(np.float32), 5)

    # 2D and 1D
    obs = (rng.random((40, 52)) * 3).astype(np.float32)
    rl_case("img2d", obs, ref.gaussian_psf((9, 9), [1.5]), 5)
    obs = (rng.random((64,)) * 3).astype(np.float32)
    k = rng.random(7)
    rl_case("sig1d", obs, (k / k.sum()).astype(np.float32), 5)

    # convergence: stop_reason == "converged"
    obs = (rng.random((8, 16, 16)) * 2 + 0.5).astype(np.float32)
    rl_case("converge", obs, ref.gaussian_psf((3, 3, 3), [0.8]), 30, rel_tol=1e-2, patience=2,
            max_iters=30)
    # rel_tol = +inf stops at patience + 1
    rl_case("tol_inf", obs, ref.gaussian_psf((3, 3, 3), [0.8]), 10, rel_tol=np.inf, patience=3,
            max_iters=10)

    # frc_resolution metric (the reference's default rule), fixed count and the
    # full default rule {frc, 1e-3, 3, 100} (deconv.hpp:35-40)
    truth = ref.generate_blobs((20, 48, 48), n_objects=4, radius_min=3, radius_max=5, seed=17,
                               noise_sigma=0.05)
    psf = ref.gaussian_psf((5, 7, 7), [1.0, 1.5, 1.5])
    frc_obs = blur_observed(truth, psf)
    rl_case("frc3d", frc_obs, psf, 6, metric="frc_resolution")
    rl_case("frc3d_default", frc_obs, psf, 100, metric="frc_resolution", rel_tol=1e-3, patience=3,
            max_iters=100)
    obs2 = (rng.random((64, 81)) * 2 + 0.2).astype(np.float32)  # odd extent: even_view trims it
    rl_case("frc2d", obs2, ref.gaussian_psf((9, 9), [1.5]), 5, metric="frc_resolution")

    # delta PSF: estimate == observed after iteration 1
    d = np.zeros((3, 3, 3), np.float32)
    d[1, 1, 1] = 1
    rl_case("delta", (rng.random((6, 10, 12)) + 0.2).astype(np.float32), d, 2)

    # rl_step (registry form, unpadded transforms; src/deconv.cpp:437-449)
    e = (rng.random((6, 14, 18)) + 0.1).astype(np.float32)
    o = (rng.random((6, 14, 18)) + 0.1).astype(np.float32)
    k = rng.random((3, 5, 5))
    k = (k / k.sum()).astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "rl_step.npz"), estimate=e, observed=o, psf=k,
                        out=ref.rl_step(e, o, k), out_accel=ref.rl_step(e, o, k, accelerated=True))

    # fft_convolve (the SPEC's unfused oracle for rl_step)
    a = rng.random((8, 8, 8)).astype(np.float32)
    kk = rng.random((3, 3, 3)).astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "fft_convolve.npz"), img=a, kernel=kk,
                        linear=ref.fft_convolve(a, kk, False),
                        circular=ref.fft_convolve(a, kk, True))

    # error cases: (kind, message) exactly as the reference raises them
    errs = {}
    good = (rng.random((4, 6, 6)) + 0.1).astype(np.float32)
    gpsf = ref.gaussian_psf((3, 3, 3), [1.0])
    neg = good.copy()
    neg[1, 2, 3] = -1e-3
    cases = {
        "rel_tol": (good, gpsf, dict(rel_tol=0.0)),
        "patience": (good, gpsf, dict(patience=0)),
        "max_iters": (good, gpsf, dict(max_iters=0)),
        "rank": (good, ref.gaussian_psf((3, 3), [1.0]), {}),
        "neg_obs": (neg, gpsf, {}),
        "neg_psf": (good, np.where(np.arange(27).reshape(3, 3, 3) == 0, -1e-4, gpsf + 1e-4 / 26)
                    .astype(np.float32), {}),
        "unnormalized": (good, (gpsf * 1.01).astype(np.float32), {}),
        "neg_both": (neg, (gpsf * 2).astype(np.float32), {}),
        "degenerate": (np.full((4, 6, 6), 0.5, np.float32), gpsf, {}),
    }
    for name, (o, k, rule) in cases.items():
        kw = dict(metric="si_psnr_vs_input", rel_tol=1e-3, patience=3, max_iters=3)
        kw.update(rule)
        try:
            ref.richardson_lucy(o, k, **kw)
            errs[name] = ("none", "")
        except ref.RefError as ex:
            errs[name] = (ex.kind, str(ex))
        np.savez_compressed(os.path.join(OUT, f"err_{name}.npz"), observed=o, psf=k,
                            kind=errs[name][0], message=errs[name][1], **{
                                f"rule_{a}": b for a, b in kw.items()})
        print("err", name, errs[name])


def gaussian_fixtures():
    """filters::gaussian (sigma 1.5, truncate 3.5: the ssim window) on 1D/2D/3D
    inputs.  The reference's metrics::ssim itself reads freed temporaries
    (it returns NaN or values > 1 here), so ssim parity is
    pinned on this filter plus the restated formula."""
    rng = np.random.default_rng(1505)
    out = {}
    for i, shp in enumerate([(64,), (40, 52), (9, 12, 15)]):
        a = (rng.random(shp) * 3).astype(np.float32)
        out[f"in{i}"] = a
        out[f"out{i}"] = ref.gaussian(a, 1.5, 3.5)
        out[f"sq{i}"] = ref.gaussian(a * a, 1.5, 3.5)
    np.savez_compressed(os.path.join(OUT, "gaussian_ssim.npz"), **out)
    print("gaussian_ssim", [v.shape for k, v in out.items() if k.startswith("in")])


def io_fixtures():
    """NDIV files written by the reference's io::write_volume, synth goldens
    (generate_blobs, gaussian_psf) and the CLI `deconvolve` pipeline run
    through the reference library (generate_blobs -> fft_convolve -> vmax 0
    -> richardson_lucy), for SURVEY.md §8(f) row f2."""
    d = os.path.join(OUT, "ndiv")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(77)
    vols = {
        "f32_zyx_spacing": (np.arange(8, dtype=np.float32).reshape(2, 2, 2), [0.29, 0.065, 0.065]),
        "f32_yx": (rng.standard_normal((5, 7)).astype(np.float32), None),
        "f32_czyx": (rng.random((3, 2, 4, 5)).astype(np.float32), [1.0, 2.5, 0.1, 0.1]),
        "u16_x": (np.array([0, 7, 65535], np.uint16), None),
        "u32_yx": (np.arange(4, dtype=np.uint32).reshape(2, 2), [1e-05, 123456789.0]),
        "bool_yx": (np.array([[1, 0], [0, 1]], np.bool_), None),
        "f32_odd_spacing": (rng.random((2, 3, 4)).astype(np.float32), [1 / 3, 2e-07, 1e16]),
    }
    man = {}
    for name, (v, sp) in vols.items():
        ref.write_volume(os.path.join(d, name + ".ndiv"), v, sp)
        man[name] = v
        man[name + "__spacing"] = np.array(sp if sp is not None else [], np.float64)
    np.savez_compressed(os.path.join(d, "manifest.npz"), **man)

    # synth goldens
    blobs = ref.generate_blobs((20, 48, 48), n_objects=6, radius_min=3.0, radius_max=4.5, seed=11,
                               noise_sigma=0.05)
    quiet = ref.generate_blobs((16, 40, 40), n_objects=3, radius_min=2.5, radius_max=4.0, seed=5,
                               noise_sigma=0.0)
    empty = ref.generate_blobs((8, 16, 16), n_objects=0, radius_min=2.0, radius_max=3.0, seed=1,
                               noise_sigma=0.05)
    psfs = {"psf_a": ref.gaussian_psf((9, 17, 17), [1.0, 2.0, 2.0]),
            "psf_b": ref.gaussian_psf((5, 5), [1.5]),
            "psf_c": ref.gaussian_psf((7,), [0.0]),
            "psf_d": ref.gaussian_psf((3, 9, 5), [0.7, 2.2, 1.1])}
    np.savez_compressed(os.path.join(OUT, "synth.npz"), blobs=blobs, quiet=quiet, empty=empty, **psfs)

    # CLI deconvolve, synthetic mode: --shape 20 48 48 --objects 4 --radius 3 4.5
    # --seed 7 --gaussian 1.0 1.5 1.5 --metric si_psnr --max-iters 6 (rel_tol 1e-3, patience 3)
    truth = ref.generate_blobs((20, 48, 48), n_objects=4, radius_min=3.0, radius_max=4.5, seed=7,
                               noise_sigma=0.05)
    ks = [2 * int(np.ceil(4.0 * s)) + 1 for s in (1.0, 1.5, 1.5)]
    psf = ref.gaussian_psf(ks, [1.0, 1.5, 1.5])
    observed = np.maximum(ref.fft_convolve(truth, psf), 0).astype(np.float32)
    r = ref.richardson_lucy(observed, psf, metric="si_psnr_vs_input", rel_tol=1e-3, patience=3,
                            max_iters=6)
    np.savez_compressed(os.path.join(OUT, "cli_synthetic.npz"), truth=truth, psf=psf, observed=observed,
                        estimate=r.estimate, metric=r.metric, iters_run=r.iters_run,
                        stop_reason=r.stop_reason, fft_shape=np.array(r.fft_shape),
                        si_blurred=ref.si_psnr(observed, truth), si_estimate=ref.si_psnr(r.estimate, truth))
    print("io fixtures", sorted(vols), blobs.shape, r.iters_run, r.stop_reason)


if __name__ == "__main__":
    if sys.argv[1:] == ["gaussian"]:
        gaussian_fixtures()
    elif sys.argv[1:] == ["io"]:
        io_fixtures()
    else:
        main()
        gaussian_fixtures()
        io_fixtures()
