"""GPU parity of filters::fft_convolve through the C
ABI: the reference's golden vectors, the numpy oracle (pinned to the
reference in test_oracle.py) on 1D/2D/3D shapes with even and odd kernels,
negative values, circular mode, and the reference's error types.  Bar: f32
relative L2 <= 1e-6 against the double-precision reference."""
import numpy as np
import pytest

from conftest import golden_files, load_golden, rel_l2
from oracle import rl_oracle as O

vk = pytest.importorskip("paper_2510_14143_b200")
pytestmark = pytest.mark.gpu

TOL = 1e-6


def test_golden_fft_convolve():
    g = load_golden(golden_files("fft_convolve")[0])
    assert rel_l2(vk.fft_convolve(g["img"], g["kernel"]), g["linear"]) <= TOL
    assert rel_l2(vk.fft_convolve(g["img"], g["kernel"], circular=True), g["circular"]) <= TOL


CASES = [
    ((64,), (7,), False), ((64,), (8,), False), ((60,), (7,), True),
    ((40, 52), (9, 9), False), ((40, 54), (4, 5), True), ((33, 47), (6, 3), False),
    ((8, 8, 8), (3, 3, 3), True), ((10, 12, 15), (3, 4, 5), True), ((16, 18, 20), (5, 6, 7), False),
    ((20, 48, 48), (7, 7, 7), False), ((5, 9, 33), (3, 3, 5), False), ((12, 30, 64), (12, 30, 64), True),
    ((64, 256, 256), (15, 15, 15), False),
]


@pytest.mark.parametrize("shape,kshape,circular", CASES, ids=lambda v: "x".join(map(str, v)) if
                         isinstance(v, tuple) else str(v))
def test_against_oracle(shape, kshape, circular):
    rng = np.random.default_rng(sum(shape) + 7 * sum(kshape))
    a = rng.standard_normal(shape).astype(np.float32)
    k = rng.standard_normal(kshape).astype(np.float32)
    want = O.fft_convolve(a, k, circular)
    got = vk.fft_convolve(a, k, circular=circular)
    assert got.shape == a.shape and got.dtype == np.float32
    assert rel_l2(got, want) <= TOL


def test_conv_plan_reuse_and_device():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    k = O.gaussian_psf((7, 7, 7), 1.2)
    plan = vk.ConvPlan((24, 40, 40), k)
    assert plan.fft_shape_ == tuple(O.good_size(s + 6) for s in (24, 40, 40))
    for s in range(3):
        a = rng.random((24, 40, 40)).astype(np.float32)
        assert rel_l2(plan.run(a), O.fft_convolve(a, k)) <= TOL
    d = torch.from_numpy(a).cuda()
    o = torch.empty_like(d)
    plan.run_device(d.data_ptr(), o.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(o.cpu().numpy(), plan.run(a))
    # a conv plan is not an RL plan
    with pytest.raises(vk.Error, match="fft_convolve"):
        lib = vk.lib()
        vk._check(lib.vk_rl_step(plan._h, a.ctypes.data, a.ctypes.data, a.ctypes.data))
    plan.close()


def test_errors_match_reference_types():
    with pytest.raises(vk.ShapeMismatch, match="ShapeMismatch: fft_convolve: rank mismatch"):
        vk.fft_convolve(np.ones((4, 4), np.float32), np.ones((3,), np.float32))
    with pytest.raises(vk.KernelTooLarge, match="KernelTooLarge: circular convolution needs kernel <= image"):
        vk.fft_convolve(np.ones((4, 4), np.float32), np.ones((5, 3), np.float32), circular=True)


@pytest.mark.parametrize("shape,kshape", [((7, 8), (3, 3)), ((7,), (7,)), ((11, 13, 14), (4, 5, 3)),
                                          ((31, 37), (31, 6)), ((9, 49, 7), (2, 1, 7))])
def test_circular_any_extent(shape, kshape):
    """Circular mode on extents the device FFT does not plan (filters.cpp:184-233:
    FFTW plans any length): periodic extension + linear convolution + crop."""
    rng = np.random.default_rng(sum(shape) * 3 + sum(kshape))
    a = rng.standard_normal(shape).astype(np.float32)
    k = rng.standard_normal(kshape).astype(np.float32)
    want = O.fft_convolve(a, k, True)
    got = vk.fft_convolve(a, k, circular=True)
    assert got.shape == a.shape
    assert rel_l2(got, want) <= TOL
    plan = vk.ConvPlan(shape, k, circular=True)
    assert np.array_equal(plan.run(a), got)
    plan.close()


def test_blur_matches_cli_synthesis():
    """observed = max(fft_convolve(truth, psf), 0) as the reference CLI builds
    it (tools/voxelkit_main.cpp:417-425), at a C1-like size."""
    import synth
    psf = O.gaussian_psf((15, 15, 15), 1.75)
    truth = synth.blobs((32, 128, 128), 10, 4.0, 8.0, seed=1)
    want = np.maximum(O.fft_convolve(truth, psf), 0)
    got = np.maximum(vk.fft_convolve(truth, psf), 0)
    assert rel_l2(got, want) <= TOL
