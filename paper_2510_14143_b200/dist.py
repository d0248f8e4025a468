"""Multi-GPU partitioning of independent volumes.

Richardson-Lucy has no exchange step between independent volumes (C3's 64
volumes, C5's 4096 fields), so the multi-GPU path is pure data partitioning:
one process per GPU, each owning a contiguous block of ceil(n/world) items
with its own plan (OTF built locally from the PSF, so no broadcast either).
torch.distributed (NCCL on the GPU box, gloo in the CPU tests) is used only
after the data path: a max-reduce of per-rank elapsed time and an all-gather
of per-rank counters.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Sequence


def shard(n_items: int, world: int, rank: int) -> range:
    """Contiguous block of items owned by `rank` (ceil(n/world) per rank; the
    tail ranks may get fewer or none)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    step = -(-n_items // world) if n_items else 0
    lo = min(rank * step, n_items)
    return range(lo, min(lo + step, n_items))


@dataclass
class RankReport:
    rank: int
    items: int
    vol_iters: int
    elapsed_s: float


def reduce_reports(local: RankReport, dist=None, device=None) -> List[RankReport]:
    """All-gather every rank's report (NCCL/gloo).  Without a process group the
    local report is returned alone."""
    if dist is None or not dist.is_initialized():
        return [local]
    import torch

    t = torch.tensor([local.rank, local.items, local.vol_iters, local.elapsed_s], dtype=torch.float64,
                     device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [RankReport(int(v[0]), int(v[1]), int(v[2]), float(v[3])) for v in (o.cpu() for o in out)]


def job_throughput(reports: Sequence[RankReport], voxels_per_item: int) -> float:
    """Whole-job voxel-iterations/s: total units over the slowest rank's time."""
    slowest = max(r.elapsed_s for r in reports)
    return sum(r.vol_iters for r in reports) * voxels_per_item / slowest if slowest > 0 else 0.0


def run_shard(items: Sequence, world: int, rank: int, work: Callable[[int, object], int]) -> RankReport:
    """Run `work(index, item) -> iterations` over this rank's block and time it
    with the host clock (callers that need device time wrap their own events)."""
    import time

    block = shard(len(items), world, rank)
    t0 = time.perf_counter()
    its = 0
    for i in block:
        its += work(i, items[i])
    return RankReport(rank, len(block), its, time.perf_counter() - t0)
