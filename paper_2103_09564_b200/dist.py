"""Multi-GPU plumbing for the brick-parallel solve.

Bricks of one pyramid level are independent ("the computation can trivially be
parallelized"), so N GPUs shard the brick batch with no data-path collective: rank r
solves bricks [r*per_rank, (r+1)*per_rank) (weak scaling).  The only communication is
the timing/metric reduction of the benchmark: max of the per-rank device time, sum of
the per-rank work.  Works with the nccl (GPU) and gloo (CPU tests) backends.
"""
from __future__ import annotations


def shard_bricks(rank: int, world: int, per_rank: int):
    """Brick ids owned by ``rank`` (contiguous, disjoint, covering world*per_rank)."""
    if not (0 <= rank < world) or per_rank < 1:
        raise ValueError("bad rank/world/per_rank")
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def reduce_metric(ms: float, work: float, device=None):
    """-> (max ms over ranks, total work over ranks).  Single process: identity."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), float(work)
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    w = torch.tensor([float(work)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t.item()), float(w.item())
