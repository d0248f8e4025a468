"""GPU side of SURVEY.md §8(f) row f2: NDIV streaming to/from device memory,
generate_blobs on the device against the reference's own output, and the
`voxelkit_b200 deconvolve` CLI against the reference pipeline
(generate_blobs -> fft_convolve -> vmax 0 -> richardson_lucy), all through
the C ABI.  Fixtures: tests/golden/{synth,cli_synthetic}.npz (make_golden.py io)."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_l2
from oracle import rl_oracle as O

vk = pytest.importorskip("paper_2510_14143_b200")
torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CLI = os.path.join(os.path.dirname(vk.LIB_PATH), "voxelkit_b200")


def test_device_stream_round_trip(tmp_path):
    """A volume larger than the 32 MiB staging chunk, odd tail included."""
    shape = (37, 301, 1003)  # 44.7 MB f32
    g = torch.Generator(device="cuda").manual_seed(3)
    d = torch.rand(shape, device="cuda", generator=g)
    p = tmp_path / "big.ndiv"
    s = torch.cuda.current_stream().cuda_stream
    vk.write_volume_device(p, d.data_ptr(), shape, np.float32, (2.0, 0.5, 0.5), stream=s)
    host = d.cpu().numpy()
    q = tmp_path / "host.ndiv"
    vk.write_volume(q, host, (2.0, 0.5, 0.5))
    assert p.read_bytes() == q.read_bytes()
    back = torch.empty_like(d)
    info = vk.read_volume_device(p, back.data_ptr(), back.numel() * 4, stream=s)
    torch.cuda.synchronize()
    assert info.shape == shape and info.spacing == (2.0, 0.5, 0.5)
    assert torch.equal(back, d)
    with pytest.raises(vk.Error, match="too small"):
        vk.read_volume_device(p, back.data_ptr(), 16, stream=s)


def _blobs(spec):
    out = torch.empty(tuple(spec.shape), device="cuda")
    sp = vk.generate_blobs_device(spec, out.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.cpu().numpy(), sp


def test_generate_blobs_matches_reference():
    g = load_golden(os.path.join(GOLDEN, "synth.npz"))
    got, sp = _blobs(vk.SynthSpec((20, 48, 48), 6, 3.0, 4.5, 11, 0.05))
    assert sp == (1.0, 1.0, 1.0)
    want = g["blobs"]
    # same mt19937_64 stream; CUDA's double log/sin/cos may differ from glibc
    # in the last ulp, which the f32 cast absorbs except at rare ties
    mism = np.count_nonzero(got != want)
    assert mism <= want.size // 10000, mism
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-6)
    quiet, _ = _blobs(vk.SynthSpec((16, 40, 40), 3, 2.5, 4.0, 5, 0.0))
    assert np.array_equal(quiet, g["quiet"])  # rasterisation alone: bit-exact
    empty, _ = _blobs(vk.SynthSpec((8, 16, 16), 0, 2.0, 3.0, 1, 0.05))
    assert np.array_equal(empty, g["empty"]) and not empty.any()
    with pytest.raises(vk.PlacementFailure, match="cannot fit the volume"):
        _blobs(vk.SynthSpec((8, 16, 16), 3, 6.0, 8.0, 1, 0.05))


def test_generate_blobs_large_is_deterministic():
    """C1-sized phantom (multiple noise chunks): deterministic, noise moments."""
    spec = vk.SynthSpec((64, 256, 256), 40, 6.0, 10.0, 1, 0.05)
    a, _ = _blobs(spec)
    b, _ = _blobs(spec)
    assert np.array_equal(a, b)
    bg = a[a < 0.5]  # mostly background: noise only
    assert abs(float(bg.std()) - 0.05) < 0.005


def _run_cli(args, cwd):
    return subprocess.run([CLI, "deconvolve", *args], cwd=cwd, capture_output=True, text=True, timeout=300)


def test_cli_synthetic_matches_reference_pipeline(tmp_path):
    g = load_golden(os.path.join(GOLDEN, "cli_synthetic.npz"))
    r = _run_cli(["--shape", "20", "48", "48", "--objects", "4", "--radius", "3", "4.5", "--seed", "7",
                  "--gaussian", "1.0", "1.5", "1.5", "--metric", "si_psnr", "--max-iters", "6",
                  "--out", str(tmp_path / "o")], tmp_path)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == f"stopped after {int(g['iters_run'])} iterations ({str(g['stop_reason'])})"
    est = vk.read_volume(tmp_path / "o" / "estimate.ndiv")
    assert est.spacing == (1.0, 1.0, 1.0)
    assert rel_l2(est.values, g["estimate"]) <= 1e-3
    summ = json.loads((tmp_path / "o" / "summary.json").read_text())
    assert summ["iters_run"] == int(g["iters_run"]) and summ["stop_reason"] == str(g["stop_reason"])
    assert summ["metric"] == "si_psnr_vs_input" and summ["schema"] == 1 and summ["backend"] == "reference"
    assert summ["fft_shape"] == [int(v) for v in g["fft_shape"]]
    np.testing.assert_allclose(summ["final_metric"], g["metric"][-1], rtol=1e-3)
    np.testing.assert_allclose(summ["si_psnr_blurred_vs_truth"], float(g["si_blurred"]), rtol=1e-4)
    np.testing.assert_allclose(summ["si_psnr_estimate_vs_truth"], float(g["si_estimate"]), rtol=1e-3)
    lines = (tmp_path / "o" / "trace.csv").read_text().splitlines()
    assert lines[0] == "iter,metric,value,wall_time_s" and len(lines) == 1 + int(g["iters_run"])
    vals = [float(line.split(",")[2]) for line in lines[1:]]
    np.testing.assert_allclose(vals, g["metric"], rtol=1e-3)


def test_cli_file_input_and_errors(tmp_path):
    psf = O.gaussian_psf((5, 7, 7), [1.0, 1.5, 1.5])
    rng = np.random.default_rng(4)
    obs = (rng.random((12, 30, 34)) * 2 + 0.1).astype(np.float32)
    vk.write_volume(tmp_path / "obs.ndiv", obs, (0.3, 0.1, 0.2))
    vk.write_volume(tmp_path / "psf.ndiv", psf)
    r = _run_cli(["--input", "obs.ndiv", "--psf", "psf.ndiv", "--metric", "frc", "--max-iters", "5",
                  "--out", "o"], tmp_path)
    assert r.returncode == 0, r.stderr
    est = vk.read_volume(tmp_path / "o" / "estimate.ndiv")
    assert est.spacing == (0.3, 0.1, 0.2)  # estimate keeps the observed's spacing
    e, t = O.richardson_lucy(obs, psf, "frc_resolution", 1e-3, 3, 5, spacing=0.2)
    assert rel_l2(est.values, e) <= 1e-3
    summ = json.loads((tmp_path / "o" / "summary.json").read_text())
    assert summ["iters_run"] == len(t.metric) and "si_psnr_blurred_vs_truth" not in summ
    # exit codes of classify() (voxelkit_main.cpp:46-66)
    assert _run_cli(["--input", "missing.ndiv", "--out", "o2"], tmp_path).returncode == 2
    (tmp_path / "junk.ndiv").write_bytes(b"JUNKJUNK")
    r = _run_cli(["--input", "junk.ndiv", "--out", "o3"], tmp_path)
    assert r.returncode == 2 and "BadMagic" in r.stderr
    neg = obs.copy()
    neg[0, 0, 0] = -1
    vk.write_volume(tmp_path / "neg.ndiv", neg)
    r = _run_cli(["--input", "neg.ndiv", "--psf", "psf.ndiv", "--out", "o4"], tmp_path)
    assert r.returncode == 5 and "NegativeInput" in r.stderr
    r = _run_cli(["--input", "obs.ndiv", "--gaussian", "1.0", "--out", "o5"], tmp_path)
    assert r.returncode == 4 and "ShapeMismatch" in r.stderr
    r = _run_cli(["--input", "obs.ndiv", "--max-iters", "0", "--out", "o6"], tmp_path)
    assert r.returncode == 2 and "max_iters must be >= 1" in r.stderr
