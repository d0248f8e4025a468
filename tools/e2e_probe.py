"""Where the end-to-end time of vk_richardson_lucy goes (pageable host arrays).

    VK_RL_TIMING=1 python tools/e2e_probe.py [c1|c2|c4|c3]

c3: the batch call on 8 volumes.  With VK_RL_TIMING=1 the library prints the
host-side phases of every vk_rl_run (h2d, run, prefault wait, d2h)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np

import bench
import paper_2510_14143_b200 as vk

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
shape = cfg["image"]
psf = bench.make_psf(*cfg["psf"], rank=len(shape))
iters = cfg["iters"]
obs = np.random.default_rng(0).random(shape, dtype=np.float32) + 0.05
rule = vk.StoppingRule("si_psnr_vs_input", 1e-300, iters, iters)

if name == "c3":
    vols = [obs + np.float32(i) * 1e-3 for i in range(8)]
    vk.richardson_lucy_batch(vols, psf, rule)
    for _ in range(3):
        t0 = time.perf_counter(); vk.richardson_lucy_batch(vols, psf, rule); t1 = time.perf_counter()
        print("batch of 8 pageable %.2f ms (%.2f per volume)" % ((t1 - t0) * 1e3, (t1 - t0) * 1e3 / 8), flush=True)
    sys.exit(0)

vk.richardson_lucy(obs, psf, rule)
for _ in range(3):
    t0 = time.perf_counter(); vk.richardson_lucy(obs, psf, rule); t1 = time.perf_counter()
    print("one-shot pageable %.2f ms" % ((t1 - t0) * 1e3), flush=True)
plan = vk.RlPlan(shape, psf)
out = np.empty_like(obs)
plan.run(obs, rule, out=out)
for _ in range(3):
    t0 = time.perf_counter(); plan.run(obs, rule, out=out); t1 = time.perf_counter()
    print("plan.run pageable, reused out %.2f ms" % ((t1 - t0) * 1e3), flush=True)
import torch

d = torch.from_numpy(obs).cuda(); do = torch.empty_like(d)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    plan.run_device(d.data_ptr(), do.data_ptr(), rule, stream=s); torch.cuda.synchronize(); t1 = time.perf_counter()
    print("device-resident %.2f ms" % ((t1 - t0) * 1e3), flush=True)
hp = torch.empty(shape, dtype=torch.float32, pin_memory=True); hp.copy_(torch.from_numpy(obs))
ho = torch.empty(shape, dtype=torch.float32, pin_memory=True)
for _ in range(3):
    t0 = time.perf_counter(); plan.run_ptr(hp.data_ptr(), ho.data_ptr(), rule); t1 = time.perf_counter()
    print("plan.run pinned %.2f ms" % ((t1 - t0) * 1e3), flush=True)
