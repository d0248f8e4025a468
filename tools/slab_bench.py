"""Cost of the §8(f4) slab decomposition on one GPU: a bench config's volume
run as 1..N in-process slabs (halo rows recomputed, halos copied after every x
pass) vs the single plan, device-resident, fixed iteration count.

    python tools/slab_bench.py c2 1,2,4
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_14143_b200 as vk  # noqa: E402
from paper_2510_14143_b200.slab import SlabPlan, copy_halos, run_slabs  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
counts = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4").split(",")]
shape, iters = cfg["image"], 10
psf = bench.make_psf(*cfg["psf"], rank=len(shape))
obs = torch.rand(shape, device="cuda") + 0.05
out = torch.empty_like(obs)
rule = vk.StoppingRule("si_psnr_vs_input", 1e-300, iters, iters)
s = torch.cuda.current_stream().cuda_stream
row = shape[1] * shape[2] * 4
ref = None
for n in counts:
    plans = [SlabPlan(shape, psf, n, r) for r in range(n)]
    ins = [obs.data_ptr() + p.image[0] * row for p in plans]
    outs = [out.data_ptr() + p.image[0] * row for p in plans]

    def go():
        return run_slabs(plans, ins, outs, psf, rule, False, lambda st: copy_halos(plans, st), lambda a, op: a, s)

    go()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        go()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / (3 * iters)
    res = out.cpu().numpy()
    if ref is None:
        ref = res
    err = float(np.linalg.norm(res - ref) / np.linalg.norm(ref))
    print(json.dumps({"config": sys.argv[1] if len(sys.argv) > 1 else "c2", "slabs": n, "ms_per_iter": round(ms, 4),
                      "rows_per_slab": [p.rows for p in plans], "rel_l2_vs_1": err}), flush=True)
    for p in plans:
        p.close()
