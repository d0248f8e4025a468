"""One volume across N GPUs: one slab plan per rank, halo
rows exchanged with the neighbours over NCCL (torch.distributed batched
isend/irecv) after every x pass, per-slab sums all-reduced.  Strong scaling
of a single-volume config; prints one JSON line on rank 0.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \\
        --master-addr 127.0.0.1 --master-port P tools/slab_dist.py --config c2
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2510_14143_b200 as vk  # noqa: E402
from paper_2510_14143_b200.slab import DistHalo, SlabPlan, dist_allreduce, run_slabs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", local))
    cfg = bench.CONFIGS[args.config]
    shape, iters = cfg["image"], cfg["iters"]
    if len(shape) != 3:
        raise SystemExit("slab decomposition is 3D only")
    psf = bench.make_psf(*cfg["psf"], rank=3)
    plan = SlabPlan(shape, psf, ws, rank, device=local)
    g = torch.Generator(device="cuda").manual_seed(1234)
    full = torch.rand(shape, device="cuda", generator=g) + 0.05  # same volume on every rank
    obs = full[plan.image[0]:plan.image[1]].contiguous()
    out = torch.empty_like(obs)
    halo = DistHalo(plan, dist, torch, psf.shape[0])
    red = dist_allreduce(dist, torch, torch.device("cuda", local))
    rule = vk.StoppingRule("si_psnr_vs_input", 1e-300, iters, iters)
    s = torch.cuda.current_stream().cuda_stream

    def step():
        return run_slabs([plan], [obs.data_ptr()], [out.data_ptr()], psf, rule, False, halo.exchange, red, s)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step()
    b.record()
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([a.elapsed_time(b)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    if rank == 0:
        n = int(np.prod(shape))
        print(json.dumps({"metric": bench.METRIC, "value": n * iters / (ms * 1e-3), "unit": bench.UNIT, "n_gpus": ws,
                          "ms_per_step": ms, "scaling": "strong",
                          "config": {"workload": cfg["label"] + f" as {ws} z slabs (one per GPU)",
                                     "rows_per_slab": plan.rows, "halo": [plan.halo_below, plan.halo_above]}}))
    plan.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
