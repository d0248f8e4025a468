"""Device ms per RL iteration under each stopping metric on a bench config
(fixed iteration count, observed image resident on the device)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_14143_b200 as vk  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
metrics = sys.argv[2].split(",") if len(sys.argv) > 2 else ["si_psnr_vs_input", "ssim_vs_prev", "frc_resolution"]
shape, iters = cfg["image"], 8
psf = bench.make_psf(*cfg["psf"], rank=len(shape))
obs = torch.rand(shape, device="cuda") + 0.05
out = torch.empty_like(obs)
plan = vk.RlPlan(shape, psf)
s = torch.cuda.current_stream().cuda_stream
for m in metrics:
    rule = vk.StoppingRule(m, 1e-300, iters, iters)
    try:
        plan.run_device(obs.data_ptr(), out.data_ptr(), rule, stream=s)
    except vk.Error as e:
        print(json.dumps({"metric": m, "error": str(e)}), flush=True)
        continue
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        plan.run_device(obs.data_ptr(), out.data_ptr(), rule, stream=s)
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"metric": m, "config": sys.argv[1] if len(sys.argv) > 1 else "c2",
                      "ms_per_iter": round(a.elapsed_time(b) / (3 * iters), 4),
                      "device_bytes": plan.device_bytes()}), flush=True)
plan.close()
