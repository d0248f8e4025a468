"""CPU: pin the numpy oracle against the reference's own outputs.

The golden fixtures were produced by the reference compiled unmodified
(tests/golden/make_golden.py); when oracle/_ref/libvkref.so is present (this
container) the oracle is also cross-checked live against it on fresh seeds.
"""
import math
import os

import numpy as np
import pytest

from conftest import golden_files, load_golden, rel_l2
from oracle import rl_oracle as O


def test_good_size_table():
    # src/fft_plan.cpp:41-49 and the FFT grids of SURVEY.md §8(a0)
    assert [O.good_size(n) for n in (0, 1, 2, 7, 11, 13, 17, 41, 97)] == [1, 1, 2, 8, 12, 15, 18, 45, 100]
    assert O.good_size(78 + 15 - 1) == 96 and O.good_size(270 + 15 - 1) == 288
    assert O.good_size(158 + 31 - 1) == 192 and O.good_size(542 + 31 - 1) == 576
    assert O.good_size(120 + 21 - 1) == 144 and O.good_size(1020 + 21 - 1) == 1080
    assert O.good_size(2078 + 31 - 1) == 2160


@pytest.mark.parametrize("path", golden_files("rl_"), ids=os.path.basename)
def test_oracle_matches_reference_goldens(path):
    if os.path.basename(path) == "rl_step.npz":
        g = load_golden(path)
        out = O.rl_step(g["estimate"], g["observed"], g["psf"])
        assert rel_l2(out, g["out"]) <= 1e-7
        assert np.array_equal(g["out"], g["out_accel"])  # reference vs accelerated backend
        return
    g = load_golden(path)
    kw = dict(metric=str(g["metric_name"]), rel_tol=float(g["rel_tol"]), patience=int(g["patience"]),
              flat_init=bool(g["flat_init"]))
    e1, t1 = O.richardson_lucy(g["observed"], g["psf"], **dict(kw, max_iters=1, patience=1))
    en, tn = O.richardson_lucy(g["observed"], g["psf"], max_iters=int(g["max_iters"]), **kw)
    assert tuple(tn.fft_shape) == tuple(int(v) for v in g["fft_shape"])
    assert rel_l2(e1, g["estimate_1"]) <= 1e-7
    assert rel_l2(en, g["estimate_n"]) <= 1e-7
    assert len(tn.metric) == int(g["iters_run"])
    assert tn.stop_reason == str(g["stop_reason"])
    np.testing.assert_allclose(tn.metric, g["metric"], rtol=1e-9)
    np.testing.assert_allclose(tn.log_likelihood, g["loglik"], rtol=1e-9)


def test_fft_convolve_golden():
    g = load_golden(golden_files("fft_convolve")[0])
    assert rel_l2(O.fft_convolve(g["img"], g["kernel"]), g["linear"]) <= 1e-7
    assert rel_l2(O.fft_convolve(g["img"], g["kernel"], True), g["circular"]) <= 1e-7


def test_ssim_gaussian_bit_exact_vs_reference():
    """The ssim window (filters::gaussian, sigma 1.5, truncate 3.5) reproduces
    the reference bit for bit, so ssim parity rests on the formula alone."""
    g = load_golden(golden_files("gaussian_ssim")[0])
    for i in range(3):
        a = g[f"in{i}"]
        assert np.array_equal(O.gaussian(a), g[f"out{i}"])
        assert np.array_equal(O.gaussian(a * a), g[f"sq{i}"])


def test_ssim_oracle_properties():
    rng = np.random.default_rng(2)
    a = (rng.random((9, 10, 11)) * 2).astype(np.float32)
    assert abs(O.ssim(a, a) - 1.0) < 1e-12
    b = (a + 0.3 * rng.random(a.shape)).astype(np.float32)
    assert 0 < O.ssim(b, a) < 1
    with pytest.raises(O.OracleError, match="ssim needs every extent >= 7"):
        O.ssim(a[:6], a[:6])


@pytest.mark.parametrize("path", golden_files("err_"), ids=os.path.basename)
def test_validation_order_and_messages(path):
    g = load_golden(path)
    kind, msg = str(g["kind"]), str(g["message"])
    kw = {k[5:]: g[k].item() for k in g if k.startswith("rule_")}
    with pytest.raises(O.OracleError) as ei:
        O.richardson_lucy(g["observed"], g["psf"], **{k: (str(v) if k == "metric" else v) for k, v in kw.items()})
    assert ei.value.kind == kind
    if kind != "UnnormalizedPsf":
        assert str(ei.value) == msg
    else:  # std::to_string(double) prints 6 decimals
        assert msg.startswith("UnnormalizedPsf: psf sums to ")
        assert abs(float(msg.split()[-1]) - float(str(ei.value).split()[-1])) < 1e-6


def test_spec_known_answers_oracle():
    rng = np.random.default_rng(3)
    # delta PSF -> estimate == observed after one iteration
    obs = (rng.random((5, 9, 11)) + 0.2).astype(np.float32)
    d = np.zeros((3, 3, 3), np.float32)
    d[1, 1, 1] = 1
    e, _ = O.richardson_lucy(obs, d, rel_tol=1e-300, patience=1, max_iters=1)
    np.testing.assert_allclose(e, obs, rtol=1e-5)
    # fixed point of the exact latent: noiseless observed = conv(truth).
    # With zero-padded 'same' convolutions the correlation of the all-ones ratio
    # is < 1 within K-1 of the border, so the fixed point holds in the interior.
    psf = O.gaussian_psf((3, 5, 5), [0.7, 1.0, 1.0])
    truth = (rng.random((10, 16, 16)) + 0.5)
    t = O.RlTransforms(truth.shape, psf)
    obs = t.convolve(truth, False)
    inner = (slice(2, -2), slice(4, -4), slice(4, -4))
    assert rel_l2(t.step(truth, obs)[inner], truth[inner]) <= 1e-4


ref = pytest.importorskip("oracle.ref")


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (make -C oracle)")
@pytest.mark.parametrize("seed,shape,kshape,flat", [
    (11, (7, 13, 17), (3, 5, 5), False), (12, (9, 10, 21), (4, 3, 6), True), (13, (33, 27), (7, 6), False),
    (14, (50,), (9,), True)])
def test_oracle_vs_reference_live(seed, shape, kshape, flat):
    rng = np.random.default_rng(seed)
    obs = (rng.random(shape) * 4).astype(np.float32)
    k = rng.random(kshape)
    k = (k / k.sum()).astype(np.float32)
    r = ref.richardson_lucy(obs, k, rel_tol=1e-300, patience=4, max_iters=4, flat_init=flat)
    e, t = O.richardson_lucy(obs, k, rel_tol=1e-300, patience=4, max_iters=4, flat_init=flat)
    assert tuple(t.fft_shape) == r.fft_shape
    assert rel_l2(e, r.estimate) <= 1e-7
    np.testing.assert_allclose(t.metric, r.metric, rtol=1e-9)
    s = ref.rl_step(obs, obs, k)
    assert rel_l2(O.rl_step(obs, obs, k), s) <= 1e-7


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (make -C oracle)")
def test_widefield_psf_properties():
    k = O.widefield_psf(31)
    assert k.shape == (31, 31, 31) and abs(float(k.astype(np.float64).sum()) - 1) < 1e-5
    assert (k >= 0).all()
    assert not np.allclose(k, k[::-1])  # axially asymmetric -> exercises the flip
    # the reference accepts it as a PSF
    obs = np.ones((4, 4, 4), np.float32) + np.arange(64, dtype=np.float32).reshape(4, 4, 4) / 64
    r = ref.richardson_lucy(obs, k, rel_tol=1e-300, patience=1, max_iters=1)
    assert r.iters_run == 1 and math.isfinite(float(r.estimate.sum()))
