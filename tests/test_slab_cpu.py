"""§8(f4) slab decomposition, host side: the decomposition math on the CPU
oracle (slabs with Kz-1-cz / cz halo rows reproduce the full run; a short halo
does not), and the neighbour exchange + all-reduce pattern of slab.DistHalo /
dist_allreduce over gloo with world size 2 (stand-in plans, CPU buffers)."""
import ctypes
import inspect
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rl_oracle as O


@pytest.mark.parametrize("kshape", [(5, 3, 3), (4, 3, 3), (7, 5, 5), (1, 3, 3)])
@pytest.mark.parametrize("nslabs", [2, 3])
def test_oracle_slabs_equal_full(kshape, nslabs):
    rng = np.random.default_rng(sum(kshape) + nslabs)
    obs = (rng.random((20, 16, 18)) * 2 + 0.1).astype(np.float32)
    k = rng.random(kshape)
    k = (k / k.sum()).astype(np.float32)
    full, _ = O.richardson_lucy(obs, k, "si_psnr_vs_input", 1e-300, 4, 4)
    np.testing.assert_allclose(O.richardson_lucy_slabs(obs, k, nslabs, 4), full, rtol=1e-6, atol=1e-7)
    full_f, _ = O.richardson_lucy(obs, k, "si_psnr_vs_input", 1e-300, 3, 3, True)
    np.testing.assert_allclose(O.richardson_lucy_slabs(obs, k, nslabs, 3, True), full_f, rtol=1e-6, atol=1e-7)


def test_short_halo_is_wrong():
    src = inspect.getsource(O.richardson_lucy_slabs).replace("hb, ha = Kz - 1 - cz, cz", "hb, ha = Kz - 2 - cz, cz")
    ns = {}
    exec(src, O.__dict__, ns)
    rng = np.random.default_rng(3)
    obs = (rng.random((20, 16, 18)) * 2 + 0.1).astype(np.float32)
    k = rng.random((5, 3, 3))
    k = (k / k.sum()).astype(np.float32)
    full, _ = O.richardson_lucy(obs, k, "si_psnr_vs_input", 1e-300, 4, 4)
    assert np.abs(ns["richardson_lucy_slabs"](obs, k, 3, 4) - full).max() > 1e-2


class _FakePlan:
    """Stand-in for SlabPlan: S_A rows as a CPU array [kx][rows][y] complex64."""

    def __init__(self, slab, nslabs, rows, own, halo_below, halo_above):
        self.slab, self.nslabs, self.rows = slab, nslabs, rows
        self.own_local = own
        self.halo_below, self.halo_above = halo_below, halo_above
        self.kx_planes, self.row_elems, self.device = 3, 5, 0
        self.S = np.zeros((self.kx_planes, rows, self.row_elems), np.complex64)

    def row_bytes(self, n):
        return self.kx_planes * n * self.row_elems * 8

    def pack(self, row, n, ptr, stream):
        blk = np.ascontiguousarray(self.S[:, row:row + n])
        ctypes.memmove(ptr, blk.ctypes.data, blk.nbytes)

    def unpack(self, row, n, ptr, stream):
        blk = np.empty((self.kx_planes, n, self.row_elems), np.complex64)
        ctypes.memmove(blk.ctypes.data, ptr, blk.nbytes)
        self.S[:, row:row + n] = blk


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_14143_b200.slab import DistHalo, dist_allreduce, halo_rows

    kz = 5
    hb, ha = halo_rows(kz)  # 2, 2
    # global P rows 0..13 split 7 / 7; slab 0 domain [0, 9), slab 1 domain [5, 14)
    if rank == 0:
        p = _FakePlan(0, 2, 9, (0, 7), 0, ha)
    else:
        p = _FakePlan(1, 2, 9, (2, 9), hb, 0)
    # owned rows carry their global row index; halos start as garbage
    q0 = 0 if rank == 0 else 5
    for r in range(p.rows):
        g = q0 + r
        own = p.own_local[0] <= r < p.own_local[1]
        p.S[:, r, :] = g if own else -1
    h = DistHalo(p, dist, torch, kz, device="cpu")
    h.exchange(0)
    ok = all((p.S[:, r, :].real == q0 + r).all() for r in range(p.rows))
    red = dist_allreduce(dist, torch, "cpu")
    s = red(np.array([1.0 + rank, 2.0]), "sum")
    mn = red(np.array([5.0 - rank]), "min")
    mx = red(np.array([5.0 - rank]), "max")
    q.put((rank, ok, s.tolist(), float(mn[0]), float(mx[0])))
    dist.destroy_process_group()


def test_dist_halo_exchange_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, True]
    assert res[0][2] == [3.0, 4.0] and res[0][3] == 4.0 and res[0][4] == 5.0
