"""GPU parity at the FULL BASELINE.json configs, on the code path bench.py
times (SURVEY.md §8(d) "Parity"): C2 128x512x512 x50, C4 100x1000x1000 x30,
C3 (two volumes of one 8-volume shard, batch lanes) and C5 (8 fields of
2048^2 x25, batch lanes).  The oracle is the reference itself
(oracle/_ref/libvkref.so: the reference's sources built unmodified, FFT =
the in-repo FFTW-API shim, double precision) on every host core.

Gates (BASELINE.json north_star): relative L2 of the f32 estimate <= 1e-4
after iteration 1 and <= 1e-3 after the final iteration; every trace value
within 1e-3 relative, log-likelihood within 1e-5.

Inputs follow SURVEY.md §8(d): the reference's generate_blobs (on the
device, bit-exact placement) blurred by fft_convolve and clamped at 0, as
the CLI builds `observed` (tools/voxelkit_main.cpp:417-425).  Both sides see
the same f32 array."""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import ref
from oracle import rl_oracle as O
import synth

vk = pytest.importorskip("paper_2510_14143_b200")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL_1, TOL_N, TOL_METRIC, TOL_LL = 1e-4, 1e-3, 1e-3, 1e-5


@pytest.fixture(autouse=True)
def _need_reference():
    if not ref.available():
        pytest.skip("oracle/_ref/libvkref.so not built")
    yield
    vk.plan_cache_clear()


def observed_3d(shape, n, seed, psf):
    torch = pytest.importorskip("torch")
    truth = torch.empty(shape, device="cuda", dtype=torch.float32)
    vk.generate_blobs_device(vk.SynthSpec(shape=tuple(shape), n_objects=n, radius_min=6.0, radius_max=10.0,
                                          seed=seed), truth.data_ptr())
    torch.cuda.synchronize()
    return np.maximum(vk.fft_convolve(truth.cpu().numpy(), psf), 0).astype(np.float32)


def observed_2d(n_side, seed, psf):
    truth = synth.blobs((n_side, n_side), 300, 6, 12, seed=seed)
    return np.maximum(vk.fft_convolve(truth, psf), 0).astype(np.float32)


def rule(iters):
    return vk.StoppingRule("si_psnr_vs_input", 1e-300, iters, iters)


def ref_run(obs, psf, iters):
    return ref.richardson_lucy(obs, psf, "si_psnr_vs_input", 1e-300, iters, iters, accelerated=True)


def check_trace(got, want):
    assert len(got.trace.records) == want.iters_run
    np.testing.assert_allclose([r.value for r in got.trace.records], want.metric, rtol=TOL_METRIC)
    np.testing.assert_allclose(got.trace.log_likelihood, want.loglik, rtol=TOL_LL)


def check_single(obs, psf, iters, expect_plan):
    plan = vk.RlPlan(obs.shape, psf)
    desc = plan.describe()
    plan.close()
    for piece in expect_plan:  # the benchmarked kernels, not the generic fallback
        assert piece in desc, desc
    r1, rn = ref_run(obs, psf, 1), ref_run(obs, psf, iters)
    g1 = vk.richardson_lucy(obs, psf, rule(1))
    gn = vk.richardson_lucy(obs, psf, rule(iters))
    assert tuple(gn.trace.fft_shape) == tuple(int(v) for v in rn.fft_shape)
    e1, en = rel_l2(g1.estimate, r1.estimate), rel_l2(gn.estimate, rn.estimate)
    print(f"relL2 iter1 {e1:.3e} iter{iters} {en:.3e}")
    assert e1 <= TOL_1 and en <= TOL_N
    check_trace(gn, rn)


def test_c2_full_config_50_iterations():
    psf = O.widefield_psf(31)
    obs = observed_3d((128, 512, 512), 600, 2, psf)
    check_single(obs, psf, 50, ["W=192x576x576", "x:fast(L=8)", "y:fast(L=8)", "z:fast(L=16)", "z:tma",
                                "y:bulk"])


def test_c4_full_config_30_iterations():
    psf = O.gaussian_psf((21, 21, 21), 2.5)
    obs = observed_3d((100, 1000, 1000), 2000, 4, psf)
    check_single(obs, psf, 30, ["W=144x1080x1080", "x:fast", "y:fast", "z:fast", "z:tma", "x:tma"])


def check_batch(vols, psf, iters, idx):
    """Volumes of one shard through the batch lanes (the bench's path); the
    estimates of `idx` against the reference, iteration 1 and the last."""
    one = vk.richardson_lucy_batch([vols[i] for i in idx], psf, rule(1))
    full = vk.richardson_lucy_batch(vols, psf, rule(iters))
    for j, i in enumerate(idx):
        r1, rn = ref_run(vols[i], psf, 1), ref_run(vols[i], psf, iters)
        e1, en = rel_l2(one[j].estimate, r1.estimate), rel_l2(full[i].estimate, rn.estimate)
        print(f"volume {i}: relL2 iter1 {e1:.3e} iter{iters} {en:.3e}")
        assert e1 <= TOL_1 and en <= TOL_N
        check_trace(full[i], rn)


def test_c3_shard_two_volumes_batch_lanes():
    """C3: a shard of 8 volumes (64 over 8 GPUs, seeds 1000..1007); its first
    and last volume against the reference."""
    psf = O.gaussian_psf((15, 15, 15), 1.75)
    vols = [observed_3d((64, 256, 256), 120, 1000 + i, psf) for i in range(8)]
    check_batch(vols, psf, 20, [0, 7])


def test_c5_eight_fields_batch_lanes():
    """C5: 8 fields of 2048^2 (the first and last two of 4 shards' worth),
    31^2 Gaussian sigma 3.75, 25 iterations, all 8 against the reference."""
    psf = O.gaussian_psf((31, 31), 3.75)
    fields = [observed_2d(2048, 5000 + i, psf) for i in range(8)]
    check_batch(fields, psf, 25, list(range(8)))
