"""Where the end-to-end time of vk_richardson_lucy goes at C2 (pageable host arrays)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2510_14143_b200 as vk
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from oracle import rl_oracle as O
shape = (128, 512, 512)
psf = O.widefield_psf(31)
obs = (np.random.default_rng(0).random(shape, dtype=np.float32) + 0.05)
rule = vk.StoppingRule("si_psnr_vs_input", 1e-300, 50, 50)
vk.richardson_lucy(obs, psf, rule)
for _ in range(3):
    t0 = time.perf_counter(); r = vk.richardson_lucy(obs, psf, rule); t1 = time.perf_counter()
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
    torch.cuda.synchronize(); t0 = time.perf_counter(); plan.run_device(d.data_ptr(), do.data_ptr(), rule, stream=s); torch.cuda.synchronize(); t1 = time.perf_counter()
    print("device-resident %.2f ms" % ((t1 - t0) * 1e3), flush=True)
hp = torch.empty(shape, dtype=torch.float32, pin_memory=True); hp.copy_(torch.from_numpy(obs))
ho = torch.empty(shape, dtype=torch.float32, pin_memory=True)
for _ in range(3):
    t0 = time.perf_counter(); plan.run_ptr(hp.data_ptr(), ho.data_ptr(), rule); t1 = time.perf_counter()
    print("plan.run pinned %.2f ms" % ((t1 - t0) * 1e3), flush=True)
