"""§8(f4) slab decomposition on the GPU: one volume split into z slabs (slab
plans in one process, halos refreshed by device copies after every x pass)
against the single-plan run of the same volume, and against the CPU oracle."""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import rl_oracle as O
import synth

vk = pytest.importorskip("paper_2510_14143_b200")
pytestmark = pytest.mark.gpu


def _rule(iters, rel_tol=1e-300, patience=None):
    return vk.StoppingRule("si_psnr_vs_input", rel_tol, patience or iters, iters)


CASES = [((40, 48, 56), (7, 5, 5), 2), ((40, 48, 56), (7, 5, 5), 3), ((33, 40, 40), (6, 5, 5), 2),
         ((64, 64, 64), (15, 15, 15), 4)]


@pytest.mark.parametrize("shape,kshape,nslabs", CASES, ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple)
                         else str(v))
def test_slabs_match_single_plan(shape, kshape, nslabs):
    from paper_2510_14143_b200.slab import richardson_lucy_slabs

    rng = np.random.default_rng(sum(shape))
    k = rng.random(kshape) + 0.3
    psf = (k / k.sum()).astype(np.float32)
    obs = synth.blurred(synth.blobs(shape, 8, 4, 7, seed=nslabs), psf) + np.float32(0.02)
    ref = vk.richardson_lucy(obs, psf, _rule(6))
    got = richardson_lucy_slabs(obs, psf, _rule(6), nslabs=nslabs)
    assert rel_l2(got.estimate, ref.estimate) <= 1e-5
    np.testing.assert_allclose([r.value for r in got.trace.records], [r.value for r in ref.trace.records], rtol=1e-5)
    np.testing.assert_allclose(got.trace.log_likelihood, ref.trace.log_likelihood, rtol=1e-6)
    its = []
    O.richardson_lucy(obs, psf, "si_psnr_vs_input", 1e-300, 6, 6, iterates=its)
    assert rel_l2(got.estimate, its[-1]) <= 1e-3


def test_slabs_flat_init_and_early_stop():
    from paper_2510_14143_b200.slab import richardson_lucy_slabs

    psf = O.gaussian_psf((5, 5, 5), 1.0)
    obs = synth.blurred(synth.blobs((30, 40, 40), 6, 4, 6, seed=3), psf) + np.float32(0.05)
    for flat in (False, True):
        ref = vk.richardson_lucy(obs, psf, _rule(30, 1e-2, 2), flat)
        got = richardson_lucy_slabs(obs, psf, _rule(30, 1e-2, 2), flat, nslabs=3)
        assert got.trace.stop_reason == ref.trace.stop_reason == "converged"
        assert len(got.trace.records) == len(ref.trace.records)
        assert rel_l2(got.estimate, ref.estimate) <= 1e-5


def test_slab_errors():
    from paper_2510_14143_b200.slab import SlabPlan, richardson_lucy_slabs

    psf = O.gaussian_psf((7, 7, 7), 1.0)
    obs = np.ones((12, 20, 20), np.float32)
    with pytest.raises(vk.Error, match="too many slabs"):
        SlabPlan(obs.shape, psf, 6, 0)
    with pytest.raises(vk.Unsupported):
        richardson_lucy_slabs(obs, psf, vk.StoppingRule("frc_resolution", 1e-3, 3, 5), nslabs=2)
    with pytest.raises(vk.DegenerateReference):
        richardson_lucy_slabs(obs, psf, _rule(3), nslabs=2)
    neg = obs.copy()
    neg[5, 3, 3] = -1
    with pytest.raises(vk.NegativeInput):
        richardson_lucy_slabs(neg, psf, _rule(3), nslabs=2)
