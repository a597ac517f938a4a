"""rw_solve_bricks_host (host buffers, H2D / solve / D2H pipelined over
chunks on separate streams): the results must equal rw_solve_bricks on the same bricks
bit for bit (each brick is solved independently with fixed-order reductions), for ragged
chunkings, pinned and pageable inputs, both solvers, and the f32 / 40^3 shapes."""
import numpy as np
import pytest
import torch

import paper_2103_09564_b200 as rwb
import workloads as wl
from gpu_helpers import dev

pytestmark = pytest.mark.gpu


def _host(a, pin):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.pin_memory() if pin else t


def _compare(p, chunk, pin, solver="auto"):
    with rwb.solver(solver):
        ref = rwb.solve_bricks(dev(p.fixed), dev(p.values), vol=dev(p.vol), beta=p.beta, eps=p.eps,
                               tol=p.tol, max_iter=p.max_iter, labels=True)
        torch.cuda.synchronize()
        got = rwb.solve_bricks_host(_host(p.fixed, pin), _host(p.values[0], pin), _host(p.vol, pin),
                                    beta=p.beta, eps=p.eps, tol=p.tol, max_iter=p.max_iter,
                                    chunk=chunk, labels=True)
    assert torch.equal(got["prob"], ref["prob"].cpu())
    assert torch.equal(got["labels"], ref["labels"].cpu())
    for k in ("iters", "resid", "status"):
        assert torch.equal(got[k], ref[k].cpu()), k


@pytest.mark.parametrize("chunk,pin", [(6, True), (0, True), (7, False), (64, True)])
def test_host_pipeline_equals_device_solve(chunk, pin):
    p = wl.cfg2(batch=20)
    _compare(p, chunk, pin)


def test_host_pipeline_streaming_solver():
    p = wl.cfg2(batch=9)
    _compare(p, 4, True, solver="streaming")


def test_host_pipeline_other_shapes():
    p = wl.cfg1()                                   # 32^3 f32, one brick
    _compare(p, 0, True)
    q = wl.random_brick(40, 40, 40, seed=3, nseed=30)
    _compare(q, 1, False)


def test_host_pipeline_rejects_device_tensors():
    p = wl.cfg2(batch=2)
    with pytest.raises(ValueError):
        rwb.solve_bricks_host(dev(p.fixed), _host(p.values[0], False), _host(p.vol, False))


def test_host_pipeline_prob_only_and_labels_only():
    p = wl.cfg2(batch=5)
    ref = rwb.solve_bricks(dev(p.fixed), dev(p.values), vol=dev(p.vol), beta=p.beta, eps=p.eps,
                           tol=p.tol, max_iter=p.max_iter, labels=True)
    torch.cuda.synchronize()
    a = rwb.solve_bricks_host(_host(p.fixed, True), _host(p.values[0], True), _host(p.vol, True),
                              beta=p.beta, eps=p.eps, tol=p.tol, max_iter=p.max_iter, chunk=2,
                              prob=True, labels=False)
    b = rwb.solve_bricks_host(_host(p.fixed, False), _host(p.values[0], False), _host(p.vol, False),
                              beta=p.beta, eps=p.eps, tol=p.tol, max_iter=p.max_iter, chunk=3,
                              prob=False, labels=True)
    assert a["labels"] is None and b["prob"] is None
    assert torch.equal(a["prob"], ref["prob"].cpu())
    assert torch.equal(b["labels"], ref["labels"].cpu())
    assert torch.equal(a["iters"], b["iters"])


@pytest.mark.parametrize("ring,chunk", [(2, 5), (4, 3)])
def test_host_streamed_ring_reuse_with_workers(ring, chunk, monkeypatch):
    """The streamed resident path with a ring of only `ring` chunk slots on a batch that
    wraps it many times, with the L2 worker clusters on (batch >= 64): every slot is refilled
    only after its previous chunk's D2H has run, so the outputs still equal the device solve."""
    monkeypatch.setenv("RW_HOST_RING", str(ring))
    p = wl.cfg2(batch=70)
    _compare(p, chunk, True)


def test_host_chunked_path_still_equal(monkeypatch):
    """The chunked path (separate launches per chunk; RW_HOST_CHUNKED=1) on a resident shape."""
    monkeypatch.setenv("RW_HOST_CHUNKED", "1")
    p = wl.cfg2(batch=20)
    _compare(p, 6, True)


def test_host_streamed_abort_falls_back(monkeypatch):
    """If a chunk's inputs never reach the persistent launch (RW_HOST_TEST_ABORT starves it,
    as a tool serialising launches would), every cluster leaves after its 2 s wait and the
    call falls back to the chunked pipeline: the results still equal the device solve."""
    monkeypatch.setenv("RW_HOST_TEST_ABORT", "1")
    p = wl.cfg2(batch=6)
    _compare(p, 2, True)
