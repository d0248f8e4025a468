#!/usr/bin/env python
"""Benchmark: Richardson-Lucy voxel-iterations/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one full Richardson-Lucy run (all of the config's iterations) over
one synthetic volume per GPU.  At N=1 the workload is BASELINE.json
configs[1] (C2: 128x512x512 float32, 31^3 widefield PSF, 50 iterations); with
N>1 every rank deconvolves its own independent volume (weak scaling, no
collective on the data path); the batch configs (c3, c5) split their volumes
across ranks in contiguous blocks (strong scaling).  `--gpus N` without a
torchrun environment re-launches itself under torch.distributed.run with N
ranks; under torchrun, --gpus must equal WORLD_SIZE.  NCCL only gathers:
the per-rank counters (all_gather) and, after the timed region, every rank's
estimates onto rank 0 (point-to-point over NVLink).

`value`   device-resident throughput: observed already in HBM, CUDA events on
          the launch stream around exactly K steps, max over ranks.
`e2e`     the same metric through the reference-facing one-shot call
          (vk_richardson_lucy / vk_richardson_lucy_batch, i.e.
          deconv::richardson_lucy[_batch]) with PAGEABLE host arrays: H2D,
          plan lookup (cached after the warm-up call), RL, D2H every step.
`roofline` SURVEY.md §8(d): the dominant KERNEL (x, y or z pass; the kinds of
          one kernel are summed) -- its algorithmic bytes (spectra, observed,
          estimate; OTF excluded, reported beside) per launch over its mean
          launch time (CUDA events around every launch, on the launch stream),
          against MEASURED_PEAKS.json hbm_gbs; `iteration_frac` = B_alg x
          voxel-iters/s per GPU / peak, B_alg = 64 S_p + 4 N_I + 8 N_P.
`cpu_baseline` the reference's own richardson_lucy (oracle/_ref, the reference
          sources built unmodified with the in-repo FFTW-API shim) on this
          host's cores, bounded sample, rank 0 at N=1.
--impl reference prints the reference arm's line (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2510_14143_b200 import dist as vdist  # noqa: E402

METRIC = "RL deconv voxel-iters/sec"
UNIT = "voxel-iters/s"

CONFIGS = {
    "c1": dict(image=(64, 256, 256), psf=("gaussian", 15, 1.75), iters=20,
               label="C1: 64x256x256 f32 volume, 15^3 Gaussian PSF (sigma 1.75), 20 RL iterations"),
    "c2": dict(image=(128, 512, 512), psf=("widefield", 31, None), iters=50,
               label="C2: 128x512x512 f32 volume, 31^3 widefield PSF, 50 RL iterations"),
    "c3": dict(image=(64, 256, 256), psf=("gaussian", 15, 1.75), iters=20, volumes=64,
               label="C3: batch of 64 volumes 64x256x256 f32, 15^3 Gaussian PSF, 20 RL iterations each"),
    "c4": dict(image=(100, 1000, 1000), psf=("gaussian", 21, 2.5), iters=30,
               label="C4: 100x1000x1000 f32 volume, 21^3 Gaussian PSF (sigma 2.5), 30 RL iterations"),
    "c5": dict(image=(2048, 2048), psf=("gaussian", 31, 3.75), iters=25,
               volumes=4096,
               label="C5: batch of 4096 fields 2048x2048 f32, 31^2 Gaussian PSF (sigma 3.75), 25 RL iterations"),
    # the paper's own deconvolution volume (reference PAPER.md:406,429: image and
    # PSF both 30x2160x2560): W = 90x6480x7680, not a BASELINE config; the CPU
    # reference would take hours per iteration and is not run (no_cpu)
    "paper": dict(image=(30, 2160, 2560), psf=("widefield_full", (30, 2160, 2560), None), iters=5, no_cpu=True,
                  e2e_steps=0,
                  label="Paper volume: 30x2160x2560 f32, same-size widefield PSF (PAPER.md:429), 5 RL iterations"),
}


def make_psf(kind, k, sigma, rank):
    """PSFs of SURVEY.md §8(d); same formulas as oracle/rl_oracle.py (restated
    here so the product bench does not import the oracle)."""
    if kind == "widefield_full":  # the widefield planes on a k = (Kz, Ky, Kx) grid
        kz, ky, kx = k
        dz = np.arange(kz, dtype=np.float64) - kz // 2
        gy = np.arange(ky, dtype=np.float64) - ky // 2
        gx = np.arange(kx, dtype=np.float64) - kx // 2
        out = np.zeros(k, np.float32)
        for i, z in enumerate(dz):
            sg = 1.5 * math.sqrt(1.0 + ((z * (1.0 + 0.15 * np.sign(z))) / 4.0) ** 2)
            plane = np.multiply.outer(np.exp(-0.5 * (gy / sg) ** 2), np.exp(-0.5 * (gx / sg) ** 2))
            out[i] = (plane / plane.sum() * math.exp(-abs(z) / 8.0)).astype(np.float32)
        return out / np.float32(out.astype(np.float64).sum())
    if kind == "widefield":
        h = k // 2
        d = np.arange(-h, h + 1, dtype=np.float64)
        out = np.zeros((k, k, k))
        for i, dz in enumerate(d):
            s = 1.5 * math.sqrt(1.0 + ((dz * (1.0 + 0.15 * np.sign(dz))) / 4.0) ** 2)
            g = np.exp(-0.5 * (d / s) ** 2)
            plane = np.multiply.outer(g, g)
            out[i] = plane / plane.sum() * math.exp(-abs(dz) / 8.0)
        return (out / out.sum()).astype(np.float32)
    d = np.arange(k, dtype=np.float64) - k // 2
    g = np.exp(-0.5 * (d / sigma) ** 2)
    v = np.ones(())
    for _ in range(rank):
        v = np.multiply.outer(v, g)
    return (v / v.sum()).astype(np.float32)


def good_size(n: int) -> int:
    """fftx::good_size (reference src/fft_plan.cpp:41-49): smallest 2^a 3^b 5^c >= n."""
    if n <= 1:
        return 1
    c = n
    while True:
        m = c
        for p in (2, 3, 5):
            while m % p == 0:
                m //= p
        if m == 1:
            return c
        c += 1


def config_dict(cfg, ws, n_batch):
    """The workload record both arms print (identical keys and values)."""
    shape, k = cfg["image"], cfg["psf"][1]
    ks = list(k) if isinstance(k, tuple) else [k] * len(shape)
    padded = [s + 2 * (kk // 2) for s, kk in zip(shape, ks)]
    return {"workload": cfg["label"] + (" per GPU" if ws > 1 and not n_batch else ""), "image": list(shape),
            "psf": ks, "iters_per_step": cfg["iters"], "volumes": n_batch or ws,
            "fft_shape": [good_size(p + kk - 1) for p, kk in zip(padded, ks)], "padded_domain": padded,
            "parallelism": (f"volume blocks over {ws} ranks" if n_batch else f"independent volumes x{ws}"),
            "l2": "inputs larger than L2" if int(np.prod(shape)) * 4 > 126e6 or n_batch else
                  "single volume partly L2-resident (126 MB L2)"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML SM clock + throttle reasons sampled every 20 ms during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.ok = False
        self.samples, self.reasons = [], set()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` outside torchrun: one rank per GPU, 127.0.0.1 rendezvous."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# kernel kinds -> the kernel that runs them (x / y / z pass)
KERNEL_OF = {"x_fwd": "xpass", "x_ratio": "xpass", "x_update": "xpass", "y_fwd": "ypass", "y_inv": "ypass",
             "y_conv": "ypass", "z_conv": "zpass", "yz_dataflow": "yzconv", "yz_cluster": "yzconv"}


def roofline(prof, otf, peak, steps):
    """Per-kernel achieved GB/s from the per-launch CUDA-event profile."""
    kern = {}
    for kind, (ms, n, alg) in prof.items():
        if not n:
            continue
        k = kern.setdefault(KERNEL_OF.get(kind, kind), {"ms": 0.0, "launches": 0, "bytes": 0, "otf_bytes": 0,
                                                        "kinds": {}})
        k["ms"] += ms
        k["launches"] += n
        k["bytes"] += alg * n
        k["otf_bytes"] += otf.get(kind, 0) * n
        k["kinds"][kind] = {"ms_per_step": round(ms / steps, 4), "launches_per_step": n // steps,
                            "alg_bytes_per_launch": alg, "otf_bytes_per_launch": otf.get(kind, 0),
                            "gbs": round(alg * n / (ms * 1e-3) / 1e9, 1) if ms else None}
    for k in kern.values():
        k["gbs"] = k["bytes"] / (k["ms"] * 1e-3) / 1e9 if k["ms"] else 0.0
        k["frac"] = k["gbs"] / peak
    return kern


def cpu_reference_run(cfg, obs, psf, iters, note):
    """The reference's richardson_lucy on the host (accelerated backend = all
    hardware threads).  Returns per-iteration wall times from its own trace."""
    from oracle import ref

    if not ref.available():
        raise FileNotFoundError("oracle/_ref/libvkref.so not built")
    r = ref.richardson_lucy(obs, psf, metric="si_psnr_vs_input", rel_tol=1e-300, patience=iters,
                            max_iters=iters, accelerated=True)
    return np.asarray(r.wall_s)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_threads():
    n = host_cores()
    env = os.environ.get("VOXELKIT_THREADS")
    if env and env.isdigit() and int(env) >= 1:
        n = min(n, int(env))
    return n


def synth_host(shape, seed):
    """Host synthetic observed volume (uniform in [0.05, 1.05): values do not
    change the work; strictly positive so no validation path triggers)."""
    rng = np.random.default_rng(seed)
    return (rng.random(shape, dtype=np.float32) + np.float32(0.05))


def run_reference_arm(args, cfg, ws, rank):
    if rank != 0:
        return
    if cfg.get("no_cpu"):
        print(json.dumps({"impl": "reference", "unavailable": "the reference on this grid takes hours per iteration"}),
              flush=True)
        return
    shape = cfg["image"]
    psf = make_psf(*cfg["psf"], rank=len(shape))
    obs = synth_host(shape, 1234)
    n_img = int(np.prod(shape))
    total = args.warmup + args.steps
    try:
        wall = cpu_reference_run(cfg, obs, psf, total, "")
        timed = wall[args.warmup:args.warmup + args.steps]
        per_it = float(np.mean(timed))
        value = n_img / per_it
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_it * 1e3,
            "higher_is_better": True, "scaling": "strong" if cfg.get("volumes") else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic", "config": config_dict(cfg, ws, cfg.get("volumes", 0)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": reference_threads(), "kind": "reference",
                             "sample": (f"one step = one RL iteration of the full {shape} volume "
                                        f"(reference richardson_lucy, accelerated backend, {total} iterations in "
                                        "one call; step time = the reference's own trace wall_time_s, "
                                        "transform setup excluded); FFT = in-repo FFTW-API shim (FFTW absent)")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
    except Exception as e:  # the oracle could not be built/loaded on this box
        line = {"impl": "reference", "unavailable": f"reference CPU build not loadable: {e}"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--volumes", type=int, default=None, help="batch size override for c3/c5")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    ws, rank, local = dist_setup(args)
    if args.impl == "ours" and "WORLD_SIZE" in os.environ and ws != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but WORLD_SIZE={ws}"}), flush=True)
        sys.exit(2)

    if args.impl == "reference":
        run_reference_arm(args, cfg, ws, rank)
        return

    import torch

    import paper_2510_14143_b200 as vk

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    shape = cfg["image"]
    iters = cfg["iters"]
    psf = make_psf(*cfg["psf"], rank=len(shape))
    n_img = int(np.prod(shape))
    # batch configs (C3 volumes, C5 fields) are split across ranks in
    # contiguous blocks (strong scaling); single-volume configs run one
    # independent volume per rank (weak scaling)
    n_batch = args.volumes if args.volumes else cfg.get("volumes", 0)
    block = vdist.shard(n_batch, ws, rank) if n_batch else range(1)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1000 + rank)
    vols = [torch.rand(shape, device="cuda", dtype=torch.float32, generator=gen) + 0.05 for _ in block]
    obs = vols[0] if vols else torch.rand(shape, device="cuda") + 0.05
    out = torch.empty_like(obs)
    plan = vk.RlPlan(shape, psf, device=local)
    rule = vk.StoppingRule(vk.StopMetric.si_psnr_vs_input, 1e-300, iters, iters)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    outs = [torch.empty_like(v) for v in vols] if n_batch else [out]
    in_ptrs, out_ptrs = [v.data_ptr() for v in vols], [o.data_ptr() for o in outs]

    def step(trace=False):
        if n_batch:  # independent volumes on the plan's concurrent batch lanes
            trs = plan.run_batch_device(in_ptrs, out_ptrs, rule, stream=sh, trace=trace)
            return trs[-1] if trs else None
        return plan.run_device(in_ptrs[0], out_ptrs[0], rule, stream=sh, trace=trace)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region -----------------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            launches += plan.launches()
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    # second timed pass of the same K steps with CUDA events around every
    # launch (on the launch stream) for the per-kernel roofline; kept out of
    # `value` because the extra event records perturb short kernels (C1)
    plan.profile(True)
    plan.profile_read(reset=True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = plan.profile_read(reset=True)
    plan.profile(False)
    t = torch.tensor([elapsed_ms], device="cuda", dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    own_ms, elapsed_ms = elapsed_ms, float(t.item())
    units_per_step = n_batch if n_batch else ws  # volumes processed by the whole job per step
    vol_iters = units_per_step * args.steps * iters
    value = vol_iters * n_img / (elapsed_ms * 1e-3)

    # ---- NCCL: per-rank counters (all_gather) -----------------------------
    mine = torch.tensor([own_ms, float(len(block) if n_batch else 1), float(iters), float(launches)],
                        device="cuda", dtype=torch.float64)
    per_rank = [mine]
    if dist:
        per_rank = [torch.empty_like(mine) for _ in range(ws)]
        dist.all_gather(per_rank, mine)
    per_rank = [[float(v) for v in t.tolist()] for t in per_rank]

    # ---- NCCL: every rank's estimates onto rank 0 (after the timed region) --
    gathered = None
    if dist:
        t0g = torch.cuda.Event(enable_timing=True)
        t1g = torch.cuda.Event(enable_timing=True)
        counts = [int(r[1]) for r in per_rank]
        t0g.record(stream)
        ops, recv = [], []
        if rank == 0:
            for src in range(1, ws):
                for _ in range(counts[src]):
                    recv.append(torch.empty_like(outs[0]))
                    ops.append(dist.P2POp(dist.irecv, recv[-1], src))
        else:
            ops = [dist.P2POp(dist.isend, o, 0) for o in outs[:counts[rank]]]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        t1g.record(stream)
        torch.cuda.synchronize()
        if rank == 0:
            gb = sum(r.numel() * 4 for r in recv)
            gathered = {"volumes": len(recv) + counts[0], "bytes_received": gb,
                        "ms": t0g.elapsed_time(t1g), "transport": "NCCL send/recv (batch_isend_irecv)"}
            del recv

    # ---- end-to-end through the reference-facing one-shot call ----------------
    # deconv::richardson_lucy[_batch] = vk_richardson_lucy[_batch]: pageable
    # numpy arrays in and out, host staging, the plan from the call's cache
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else cfg.get("e2e_steps", max(1, min(args.steps, 5)))
    e2e_value = None
    e2e_vols = 0
    first_call_ms = None
    if e2e_steps > 0:
        # batch configs: at most 64 volumes per rank (pageable host memory for
        # the whole C5 block would be 2 x 69 GB)
        e2e_src = vols[-64:] if n_batch else [vols[-1]]
        host_in = [v.cpu().numpy() for v in e2e_src]  # pageable
        e2e_vols = len(host_in)

        def e2e_call():
            if n_batch:
                return [r.estimate for r in vk.richardson_lucy_batch(host_in, psf, rule, device=local)]
            return [vk.richardson_lucy(host_in[0], psf, rule, device=local).estimate]

        tc = time.perf_counter()
        e2e_call()  # warm: builds and caches the plan
        first_call_ms = (time.perf_counter() - tc) * 1e3
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = e2e_call()
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_value = ws * e2e_vols * e2e_steps * iters * n_img / float(te.item())
        assert np.array_equal(res[-1], outs[(len(block) - 1) if n_batch else 0].cpu().numpy()), \
            "host-API and device-API results differ"
        del res
        vk.plan_cache_clear()

    # ---- roofline of the dominant kernel -------------------
    peak, peak_src = load_peaks()
    kern = roofline(prof, plan.otf_bytes(), peak, args.steps)
    dom = max(kern, key=lambda k: kern[k]["ms"])
    kd = kern[dom]
    g = plan.fft_shape_
    P = plan.domain_shape
    pz, py = (P[-3] if len(P) == 3 else 1), (P[-2] if len(P) >= 2 else 1)
    hx = g[-1] // 2 + 1
    s_p = pz * py * hx
    b_alg = 64 * s_p + 4 * n_img + 8 * int(np.prod(P))
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get("per_kernel", {}).get(dom, {}).get("dram_bytes_per_launch")
    kernel_total_ms = sum(k["ms"] for k in kern.values())
    vox_it_per_gpu = value / ws
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if n_batch else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, ws, n_batch),
        "plan": {"describe": plan.describe(), "fft_shape": list(g), "padded_domain": list(P),
                 "spectrum_mb": round(s_p * 8 / 1e6, 1), "observed_mb": round(n_img * 4 / 1e6, 1)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": kd["gbs"], "peak": peak, "unit": "GB/s",
                     "frac": kd["frac"], "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": kd["bytes"] / kd["launches"],
                     "mean_launch_ms": kd["ms"] / kd["launches"],
                     "kernel_share_of_step": kd["ms"] / kernel_total_ms if kernel_total_ms else None,
                     "bytes": "SURVEY.md §8(d): spectra + observed + estimate; OTF excluded (otf_bytes_per_launch)",
                     "timing": "CUDA events around every launch on the launch stream, second timed pass of the "
                               "same K steps",
                     "per_kernel": {k: {"ms_per_step": round(v["ms"] / args.steps, 4), "gbs": round(v["gbs"], 1),
                                        "frac": round(v["frac"], 4), "kinds": v["kinds"]} for k, v in kern.items()},
                     "iteration_B_alg_bytes": b_alg,
                     "iteration_frac": vox_it_per_gpu / n_img * b_alg / 1e9 / peak},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": e2e_vols * n_img * 4,
                "d2h_bytes_per_step": e2e_vols * (n_img * 4 + iters * 3 * 8), "bytes_scope": "per rank",
                "api": ("vk_richardson_lucy_batch (deconv::richardson_lucy_batch)" if n_batch
                        else "vk_richardson_lucy (deconv::richardson_lucy)")
                       + ": pageable host arrays, pinned staging ring, cached plan",
                "first_call_ms": first_call_ms,
                "first_call": "the untimed warm-up call: plan creation (device buffers, both OTFs, their "
                              "symmetry / rank-1 tests) + the same run; the timed calls reuse the cached plan",
                "volumes_per_rank": e2e_vols, "steps": e2e_steps},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "per_rank": [{"rank": i, "elapsed_ms": r[0], "volumes": int(r[1]), "iters": int(r[2]),
                      "launches": int(r[3])} for i, r in enumerate(per_rank)],
    }
    if gathered:
        line["results_gather"] = gathered
    if rank == 0 and ws == 1 and cfg.get("no_cpu"):
        line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "reference",
                                "sample": "not run: the reference on this grid takes hours per iteration"}
    elif rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            host_obs = obs.cpu().numpy()
            t0 = time.perf_counter()
            wall = cpu_reference_run(cfg, host_obs, psf, 2, "")
            per_it = float(wall[-1])
            line["cpu_baseline"] = {
                "value": n_img / per_it, "unit": UNIT, "cores": reference_threads(), "kind": "reference",
                "sample": (f"reference richardson_lucy (sources built unmodified, in-repo FFTW-API shim) on the "
                           f"same {shape} volume and PSF, 2 iterations, accelerated backend; value from the "
                           f"steady-state iteration's trace wall_time_s ({per_it:.2f} s); call took "
                           f"{time.perf_counter() - t0:.1f} s")}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
