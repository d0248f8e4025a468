"""Sweep the dataflow lag/ring (env VK_RL_DF_LAG / VK_RL_DF_RING) on a config
and print per-kernel device ms per iteration (CUDA events around launches)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_14143_b200 as vk  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
settings = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{}]
shape, iters = cfg["image"], 10
psf = bench.make_psf(*cfg["psf"], rank=len(shape))
obs = torch.rand(shape, device="cuda") + 0.05
out = torch.empty_like(obs)
rule = vk.StoppingRule("si_psnr_vs_input", 1e-300, iters, iters)
for env in settings:
    for k in ("VK_RL_DF_LAG", "VK_RL_DF_RING", "VK_RL_NO_DATAFLOW", "VK_RL_NO_L2_PERSIST"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    plan = vk.RlPlan(shape, psf)
    s = torch.cuda.current_stream().cuda_stream
    plan.run_device(obs.data_ptr(), out.data_ptr(), rule, stream=s)
    plan.profile(True)
    plan.profile_read(reset=True)
    for _ in range(3):
        plan.run_device(obs.data_ptr(), out.data_ptr(), rule, stream=s)
    torch.cuda.synchronize()
    prof = plan.profile_read(reset=True)
    per_it = {k: round(v[0] / (3 * iters), 4) for k, v in prof.items() if v[1]}
    print(json.dumps({"env": env, "plan": plan.describe(), "ms_per_iter": per_it,
                      "total": round(sum(per_it.values()), 4)}), flush=True)
    plan.close()
