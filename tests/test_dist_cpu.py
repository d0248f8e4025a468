"""CPU: the multi-GPU partitioning logic with world_size 2 over gloo.

Each rank deconvolves its contiguous block of independent volumes (here with
the numpy oracle standing in for the device, since this container has no
GPU), the reports are all-gathered, and the union must equal a single-process
run volume by volume (no exchange step exists between volumes)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_14143_b200 import dist as vdist


def test_shard_partition_properties():
    for n in (0, 1, 7, 64, 4096, 65):
        for world in (1, 2, 3, 4, 8):
            blocks = [vdist.shard(n, world, r) for r in range(world)]
            flat = [i for b in blocks for i in b]
            assert flat == list(range(n))  # disjoint, complete, ordered
            sizes = [len(b) for b in blocks]
            assert max(sizes, default=0) - min(sizes, default=0) <= -(-n // world)
    assert list(vdist.shard(64, 8, 3)) == list(range(24, 32))  # C3: 8 volumes per GPU
    assert len(vdist.shard(4096, 8, 7)) == 512  # C5: 512 fields per GPU
    with pytest.raises(ValueError):
        vdist.shard(4, 2, 2)


def test_job_throughput_uses_slowest_rank():
    reps = [vdist.RankReport(0, 2, 40, 1.0), vdist.RankReport(1, 2, 40, 2.0)]
    assert vdist.job_throughput(reps, 100) == 80 * 100 / 2.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _volumes():
    rng = np.random.default_rng(0)
    from oracle import rl_oracle as O

    psf = O.gaussian_psf((3, 5, 5), [0.8, 1.2, 1.2])
    vols = [(rng.random((4, 10, 12)) + 0.1).astype(np.float32) for _ in range(5)]
    return vols, psf


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import rl_oracle as O

    vols, psf = _volumes()
    results = {}

    def work(i, v):
        e, t = O.richardson_lucy(v, psf, "si_psnr_vs_input", 1e-300, 3, 3)
        results[i] = e
        return len(t.metric)

    rep = vdist.run_shard(vols, world, rank, work)
    reports = vdist.reduce_reports(rep, dist)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), idx=np.array(sorted(results)),
             est=np.stack([results[i] for i in sorted(results)]) if results else np.zeros((0, 4, 10, 12)),
             reports=np.array([[r.rank, r.items, r.vol_iters, r.elapsed_s] for r in reports]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_partition_matches_single_process(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    from oracle import rl_oracle as O

    vols, psf = _volumes()
    seen = []
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        rep = z["reports"]
        assert rep.shape == (world, 4)
        assert list(rep[:, 0]) == [0, 1] and int(rep[:, 1].sum()) == len(vols)
        assert int(rep[:, 2].sum()) == 3 * len(vols)
        for i, e in zip(z["idx"], z["est"]):
            ref, _ = O.richardson_lucy(vols[i], psf, "si_psnr_vs_input", 1e-300, 3, 3)
            np.testing.assert_array_equal(e, ref)
            seen.append(int(i))
    assert sorted(seen) == list(range(len(vols)))
