"""GPU: the multi-rank partition through the real C ABI.

Two processes share cuda:0 over gloo (this run has one GPU; NCCL over NVLink
takes gloo's place on a multi-GPU box).  Each rank deconvolves its
contiguous block of independent volumes through vk_richardson_lucy_batch,
the per-rank counters are all-gathered and the estimates are gathered onto
rank 0 with point-to-point sends, as bench.py does.  The union must equal a
single-process batch run bit for bit (volumes never exchange data)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPE, N_VOL, ITERS = (12, 40, 36), 5, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    from oracle import rl_oracle as O

    rng = np.random.default_rng(3)
    psf = O.gaussian_psf((5, 5, 5), 1.0)
    vols = [(rng.random(SHAPE) + 0.1).astype(np.float32) for _ in range(N_VOL)]
    return vols, psf


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import paper_2510_14143_b200 as vk
    from paper_2510_14143_b200 import dist as vdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    vols, psf = _inputs()
    block = vdist.shard(len(vols), world, rank)
    rule = vk.StoppingRule("si_psnr_vs_input", 1e-300, ITERS, ITERS)
    res = vk.richardson_lucy_batch([vols[i] for i in block], psf, rule) if len(block) else []
    rep = vdist.reduce_reports(vdist.RankReport(rank, len(block), ITERS * len(block), 0.0), dist)
    counts = [r.items for r in rep]
    if rank == 0:
        got = [torch.from_numpy(r.estimate) for r in res]
        for src in range(1, world):
            for _ in range(counts[src]):
                t = torch.empty(SHAPE, dtype=torch.float32)
                dist.recv(t, src)
                got.append(t)
        np.save(os.path.join(out_dir, "gathered.npy"), torch.stack(got).numpy())
    else:
        for r in res:
            dist.send(torch.from_numpy(r.estimate), 0)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_through_the_c_abi_match_one_process(tmp_path):
    import paper_2510_14143_b200 as vk

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    vols, psf = _inputs()
    rule = vk.StoppingRule("si_psnr_vs_input", 1e-300, ITERS, ITERS)
    single = np.stack([r.estimate for r in vk.richardson_lucy_batch(vols, psf, rule)])
    gathered = np.load(tmp_path / "gathered.npy")
    assert gathered.shape == single.shape
    assert np.array_equal(gathered, single)
