"""CPU: the C-ABI library loads, exports every symbol include/vk_rl.h declares,
and validates arguments in the reference's order before touching a GPU."""
import ctypes

import numpy as np
import pytest

import paper_2510_14143_b200 as vk
from oracle import rl_oracle as O


def test_header_symbols_exported():
    names = vk.exported_symbols()
    assert len(names) >= 14
    L = vk.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.vk_abi_version() == 4


def test_good_size_matches_oracle():
    for n in list(range(0, 200)) + [1079, 1081, 2077, 2159, 4097]:
        assert vk.good_size(n) == O.good_size(n)


def _rule(**kw):
    base = dict(metric=vk.StopMetric.si_psnr_vs_input, rel_tol=1e-3, patience=3, max_iters=3)
    base.update(kw)
    return vk.StoppingRule(**base)


@pytest.mark.parametrize("kw,msg", [
    (dict(rel_tol=0.0), "rel_tol must be positive"),
    (dict(rel_tol=-1.0), "rel_tol must be positive"),
    (dict(patience=0), "patience must be >= 1"),
    (dict(max_iters=0), "max_iters must be >= 1"),
])
def test_rule_validation_before_gpu(kw, msg):
    obs = np.ones((4, 5, 6), np.float32)
    psf = O.gaussian_psf((3, 3, 3), [1.0])
    with pytest.raises(vk.Error) as ei:
        vk.richardson_lucy(obs, psf, _rule(**kw))
    assert type(ei.value) is vk.Error and str(ei.value) == msg


def test_rank_mismatch_before_gpu():
    obs = np.ones((4, 5, 6), np.float32)
    with pytest.raises(vk.ShapeMismatch) as ei:
        vk.richardson_lucy(obs, O.gaussian_psf((3, 3), [1.0]), _rule())
    assert str(ei.value) == "ShapeMismatch: psf rank must match the image rank"
    with pytest.raises(vk.ShapeMismatch):
        vk.RlTransforms((4, 5, 6), O.gaussian_psf((3, 3), [1.0]))


def test_rl_step_shape_errors_before_gpu():
    with pytest.raises(vk.ShapeMismatch) as ei:
        vk.rl_step(np.ones((3, 4)), np.ones((3, 5)), O.gaussian_psf((3, 3), [1.0]))
    assert str(ei.value) == "ShapeMismatch: rl_step: [3,4] vs [3,5]"


def test_negative_infinite_tol_passes_rule_check():
    # -inf passes the reference's rule check (isinf), so the failure comes later
    # (here: no GPU / or a real run) and is not the rel_tol error.
    obs = np.ones((4, 5, 6), np.float32)
    psf = O.gaussian_psf((3, 3, 3), [1.0])
    try:
        vk.richardson_lucy(obs, psf, _rule(rel_tol=-np.inf))
    except vk.Error as e:
        assert "rel_tol" not in str(e)


def test_trace_csv_format():
    t = vk.IterationTrace([vk.IterationRecord(1, "si_psnr_vs_input", 12.5, 0.25),
                           vk.IterationRecord(2, "frc_resolution", float("inf"), 0.5)])
    assert t.to_csv() == "iter,metric,value,wall_time_s\n1,si_psnr_vs_input,12.5,0.25\n2,frc_resolution,inf,0.5\n"


def test_bench_roofline_groups_kinds_by_kernel():
    """bench.py's §8(d) roofline: kinds of one kernel are summed, OTF bytes are
    reported beside the algorithmic bytes and never inside them."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    prof = {"x_ratio": (10.0, 10, 500), "x_update": (20.0, 10, 900), "z_conv": (25.0, 20, 400),
            "y_fwd": (1.0, 0, 0)}
    k = bench.roofline(prof, {"z_conv": 256}, peak=1.0, steps=10)
    assert set(k) == {"xpass", "zpass"}
    assert k["xpass"]["bytes"] == 10 * 500 + 10 * 900 and k["xpass"]["ms"] == 30.0
    assert abs(k["xpass"]["gbs"] - (14000 / 0.030) / 1e9) < 1e-12
    assert k["zpass"]["otf_bytes"] == 20 * 256 and k["zpass"]["bytes"] == 20 * 400


def test_bench_config_records_match_the_reference_rules():
    """Both bench arms print the same config dict; its fft_shape / padded
    domain follow the reference's rules (deconv.cpp:114-116, 210-219) and
    SURVEY.md §8(a0)."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for n in list(range(0, 300)) + [2077, 6479, 7679]:
        assert bench.good_size(n) == O.good_size(n)
    want = {"c1": ([78, 270, 270], [96, 288, 288]), "c2": ([158, 542, 542], [192, 576, 576]),
            "c4": ([120, 1020, 1020], [144, 1080, 1080]), "c5": ([2078, 2078], [2160, 2160])}
    for name, (padded, fft) in want.items():
        cfg = bench.CONFIGS[name]
        d = bench.config_dict(cfg, 1, cfg.get("volumes", 0))
        assert d["padded_domain"] == padded and d["fft_shape"] == fft
        assert d == bench.config_dict(cfg, 1, cfg.get("volumes", 0))
