"""World-size-2 CPU (gloo) test of the N>1 host path: brick sharding and the timing/work
reduction bench.py uses.  Each rank solves its shard with the oracle (CPU)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2103_09564_b200.dist import shard_bricks, reduce_metric


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import workloads as wl
    from oracle import rw_oracle as ro
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    ids = shard_bricks(rank, world, 2)
    p = wl.cfg2(bricks=ids, n=16)
    o = ro.solve_problem(p, tol=1e-6)
    work = float(o["iters"].sum()) * 16 ** 3
    ms = 10.0 + rank                       # synthetic per-rank time: max must be 11
    mx, tot = reduce_metric(ms, work)
    out[rank] = (ids, work, mx, tot)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_reduction():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    ids0, w0, mx0, tot0 = out[0]
    ids1, w1, mx1, tot1 = out[1]
    assert sorted(ids0 + ids1) == list(range(4)) and not set(ids0) & set(ids1)
    assert mx0 == mx1 == 11.0
    assert tot0 == tot1 == w0 + w1
    # the sum over shards equals the single-process solve of all four bricks
    import workloads as wl
    from oracle import rw_oracle as ro
    o = ro.solve_problem(wl.cfg2(bricks=range(4), n=16), tol=1e-6)
    assert np.isclose(tot0, float(o["iters"].sum()) * 16 ** 3)


def test_single_process_reduce_is_identity():
    assert reduce_metric(3.5, 7.0) == (3.5, 7.0)
    assert shard_bricks(1, 4, 3) == [3, 4, 5]
