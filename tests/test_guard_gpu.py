"""Out-of-bounds-write checks without compute-sanitizer (closed on this GPU
pool): every device buffer a plan allocates carries guard bands
(VK_RL_GUARD=1, vk_debug_guard_check), and caller-owned device outputs are
checked with canaries around them."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2510_14143_b200 as vk
import synth
from oracle import rl_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_plan_buffers_guard_bands_intact():
    """Every kernel family (fast x/y/z passes at the configs' lengths with
    TMA / bulk copies, the kx-chunk ring, generic Stockham, FRC / SSIM,
    device-side stopping, batch lanes, fft_convolve, rl_step) runs with
    64 KB guard bands around each plan buffer; none may be overwritten."""
    env = dict(os.environ, VK_RL_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), "small"], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "SANITIZE_CASES_DONE" in r.stdout, r.stdout[-2000:]
    assert "GUARD_VIOLATIONS 0" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
    assert "vk guard:" not in r.stderr, r.stderr[-4000:]


@pytest.mark.parametrize("shape,kshape", [((24, 80, 72), (9, 9, 9)), ((128, 512, 60), (31, 31, 31)),
                                          ((300, 260), (31, 31))])
def test_device_output_canaries(shape, kshape):
    """run_device writes exactly the image extent of the caller's buffer:
    canaries on both sides of the output stay untouched (estimate crop, the
    UPDATE_LAST x pass writing the output directly)."""
    import torch

    psf = O.widefield_psf(kshape[0]) if len(shape) == 3 and kshape[0] == 31 else \
        O.gaussian_psf(kshape, 1.5)
    obs = synth.blurred(synth.blobs(shape, 12, 4, 7, seed=3), psf) if len(shape) == 3 else \
        (np.random.default_rng(1).random(shape) + 0.1).astype(np.float32)
    n = obs.size
    pad = 1 << 16
    big = torch.full((n + 2 * pad,), float("nan"), device="cuda", dtype=torch.float32)
    canary = big[:pad].clone()
    d_obs = torch.from_numpy(obs).cuda()
    plan = vk.RlPlan(obs.shape, psf)
    for rule in (vk.StoppingRule("si_psnr_vs_input", 1e-300, 3, 3), vk.StoppingRule("si_psnr_vs_input", 1e-2, 2, 6)):
        plan.run_device(d_obs.data_ptr(), big[pad:pad + n].data_ptr(), rule,
                        stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        lo, hi = big[:pad], big[pad + n:]
        assert torch.isnan(lo).all() and torch.isnan(hi).all(), "write outside the output extent"
        assert torch.equal(lo.view(torch.int32), canary.view(torch.int32))
        assert torch.isfinite(big[pad:pad + n]).all()
    plan.close()
