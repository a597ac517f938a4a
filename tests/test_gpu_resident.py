"""GPU parity of the brick-resident solver (one thread-block cluster per brick, CG state on
chip; include/rw.h "Solver selection") against the fp64 oracle, and its
agreement with the streaming solver.  Same bars as test_gpu_parity.py (BASELINE.json
north_star): |dp| <= 1e-4, labels exact outside the 1e-3 band.
"""
import numpy as np
import pytest
import torch

import paper_2103_09564_b200 as rwb
import workloads as wl
from oracle import rw_oracle as ro
from paper_2103_09564_b200._lib import RWError
from gpu_helpers import gpu_solve, assert_prob_parity, assert_label_parity

pytestmark = pytest.mark.gpu


def resident(p, **kw):
    with rwb.solver("resident"):
        return gpu_solve(p, **kw)


def streaming(p, **kw):
    with rwb.solver("streaming"):
        return gpu_solve(p, **kw)


def test_resident_available_shapes():
    assert rwb.resident_available((64, 64, 64))
    assert rwb.resident_available((32, 32, 32))
    assert rwb.resident_available((40, 40, 40))       # the paper's s_e = 1.25 * 32
    assert rwb.resident_available((64, 64, 64), nrhs=3)   # (rhs, brick) pairs
    assert not rwb.resident_available((48, 48, 48))
    p = wl.random_brick(48, 8, 8, seed=1, nseed=10)
    with rwb.solver("resident"), pytest.raises(RWError, match="RW_EUNSUPPORTED"):
        gpu_solve(p)


def test_cfg1_resident_parity():
    p = wl.cfg1()
    o = resident(p)
    ref = ro.solve_problem(p, tol=1e-10)
    assert_prob_parity(o["prob"], ref["prob"])
    assert_label_parity(o["labels"], ref["prob"][0])
    assert o["status"][0, 0] == 1 and o["resid"][0, 0] <= 1e-6
    it_o = ro.solve_problem(p, tol=1e-6)["iters"][0, 0]
    assert abs(int(o["iters"][0, 0]) - int(it_o)) <= 5, (o["iters"], it_o)


def test_cfg2_resident_parity_batch_invariance_and_streaming_agreement():
    ids = [0, 37, 101, 150, 199, 255, 300, 333, 377, 400, 421, 450, 470, 490, 500, 511]
    p = wl.cfg2(bricks=ids)
    o = resident(p)
    for j in (0, 5, 15):
        ref = ro.solve_problem(p, tol=1e-10, bricks=[j])
        assert_prob_parity(o["prob"][:, j:j + 1], ref["prob"])
        assert_label_parity(o["labels"][j], ref["prob"][0, 0])
    # a brick's bits do not depend on the batch or on which cluster solved it
    alone = resident(p.subset([5]))
    assert np.array_equal(alone["prob"][0, 0], o["prob"][0, 5])
    assert alone["iters"][0, 0] == o["iters"][0, 5]
    assert (o["status"] == 1).all() and (o["iters"] > 100).all()
    s = streaming(p)
    assert np.abs(s["prob"] - o["prob"]).max() <= 2e-5
    assert np.abs(s["iters"].astype(int) - o["iters"].astype(int)).max() <= 3
    np.testing.assert_allclose(s["resid"], o["resid"], rtol=0.05)


@pytest.mark.parametrize("n", [32, 40, 64])
def test_resident_random_bricks_many_per_cluster(n):
    """More bricks than co-resident clusters (each cluster solves several), random seeds with
    continuous values; u16 intensities.  n = 40 has idle lanes (10 quads per row)."""
    batch = {32: 40, 40: 40, 64: 10}[n]
    p = wl.random_brick(n, n, n, seed=100 + n, batch=batch, nseed=n ** 3 // 60,
                        continuous=True, dtype="u16")
    o = resident(p, tol=1e-7, max_iter=20000)
    s = streaming(p, tol=1e-7, max_iter=20000)
    assert (o["status"] == 1).all()
    assert np.abs(s["prob"] - o["prob"]).max() <= 2e-5
    for j in (0, batch - 1):
        ref = ro.solve_problem(p, tol=1e-11, bricks=[j])
        assert_prob_parity(o["prob"][:, j:j + 1], ref["prob"])


@pytest.mark.parametrize("n", [32, 40])
def test_resident_wide_shape(n):
    """RW_OPT_RESIDENT_WIDE (10- / 8-CTA clusters of 4 planes for 40^3 / 32^3) against the
    oracle and the default 5- / 4-CTA shape; batch invariance within the wide shape."""
    p = wl.random_brick(n, n, n, seed=200 + n, batch=6, nseed=n ** 3 // 60, continuous=True,
                        dtype="u16")
    d = resident(p, tol=1e-7, max_iter=20000)
    rwb.set_resident_wide(True)
    try:
        w = resident(p, tol=1e-7, max_iter=20000)
        one = resident(p.subset([4]), tol=1e-7, max_iter=20000)
    finally:
        rwb.set_resident_wide(False)
    assert (w["status"] == 1).all()
    assert np.abs(w["prob"] - d["prob"]).max() <= 2e-5
    assert np.abs(w["iters"].astype(int) - d["iters"].astype(int)).max() <= 2
    assert np.array_equal(one["prob"][0, 0], w["prob"][0, 4])
    ref = ro.solve_problem(p, tol=1e-11, bricks=[0])
    assert_prob_parity(w["prob"][:, 0:1], ref["prob"])


def test_resident_degenerate_bricks():
    """As test_degenerate_bricks on 32^3: no fixed voxel -> TRIVIAL 0.5; all fixed ->
    TRIVIAL values; all fixed values 0 -> ZERO_B; a normal brick vs the oracle."""
    p = wl.random_brick(32, 32, 32, seed=9, batch=4, nseed=300)
    p.fixed[0] = 0
    p.fixed[1] = 1
    p.values[0, 1] = np.random.default_rng(0).uniform(0, 1, p.values[0, 1].shape)
    p.values[0, 2] = 0.0
    o = resident(p, tol=1e-7)
    assert o["status"][0].tolist()[:3] == [3, 3, 4]
    assert o["iters"][0].tolist()[:3] == [0, 0, 0]
    assert np.all(o["prob"][0, 0] == 0.5)
    np.testing.assert_array_equal(o["prob"][0, 1], p.values[0, 1])
    assert np.all(o["prob"][0, 2] == 0.0)
    ref = ro.solve_problem(p.subset([3]), tol=1e-11)
    assert_prob_parity(o["prob"][:, 3:4], ref["prob"])
    s = streaming(p, tol=1e-7)
    assert np.array_equal(s["status"], o["status"])


def test_resident_max_iter_abs_mode_warm_start_and_W():
    p = wl.random_brick(32, 32, 32, seed=11, nseed=200)
    o = resident(p, tol=1e-12, max_iter=3)
    assert o["iters"][0, 0] == 3 and o["status"][0, 0] == 2
    s = streaming(p, tol=1e-12, max_iter=3)
    assert np.abs(s["prob"] - o["prob"]).max() <= 1e-6
    ref = ro.solve_problem(p, tol=1e-11)
    a = resident(p, tol=1e-3, tol_mode=1)
    assert a["status"][0, 0] == 1 and a["resid"][0, 0] <= 1e-3
    w = resident(p, tol=1e-6, x0=ref["x"].astype(np.float32))
    assert w["iters"][0, 0] <= 3
    v = resident(p)
    u = resident(p, use_W=True)
    assert np.array_equal(v["prob"], u["prob"]) and np.array_equal(v["iters"], u["iters"])


def test_cosched_matches_resident_only():
    """RW_OPT_COSCHED (include/rw.h): the last share of a 64^3 batch runs through the
    streaming passes on a second stream next to the resident clusters.  Results agree with
    the resident-only solve to the solver tolerance, iteration counts within 3."""
    from paper_2103_09564_b200._lib import lib
    ids = list(range(0, 512, 4))
    p = wl.cfg2(bricks=ids)
    a = resident(p)
    old = lib().rw_get_option(1)
    lib().rw_set_option(1, 250)
    try:
        ws = rwb.api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, p.dims, 1) * 2, "cuda")
        b = gpu_solve(p, workspace=ws)
    finally:
        lib().rw_set_option(1, old)
    assert (b["status"] == 1).all()
    assert np.abs(a["prob"] - b["prob"]).max() <= 2e-5
    assert np.abs(a["iters"].astype(int) - b["iters"].astype(int)).max() <= 3
    nres = len(ids) - len(ids) * 250 // 1000
    assert np.array_equal(a["prob"][:, :nres], b["prob"][:, :nres])     # resident part bitwise


@pytest.mark.parametrize("n", [32, 40, 64])
def test_resident_multilabel_parity(n):
    """rw_solve_labels on the resident solver (K-1 = 3 rhs as (rhs, brick) pairs on one
    operator) against K explicit fp64 oracle solves (reading R11)."""
    lp = wl.cfg4(n=n, seeds_per_label=max(20, n // 2))
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    outs = {}
    for name in ("resident", "streaming"):
        with rwb.solver(name):
            o = rwb.solve_labels(dv(lp.labels), lp.K, vol=dv(lp.vol), beta=lp.beta, eps=lp.eps,
                                 tol=lp.tol, max_iter=lp.max_iter)
        torch.cuda.synchronize()
        outs[name] = {k: v.cpu().numpy() for k, v in o.items() if v is not None}
    prob, lab = outs["resident"]["prob"], outs["resident"]["labels"]
    ref = ro.solve_labels(lp, tol=1e-10)
    assert_prob_parity(prob, ref["prob"][: lp.K - 1])
    derived = np.clip(1.0 - prob.astype(np.float64).sum(axis=0), 0, 1)
    assert np.abs(derived - ref["prob"][lp.K - 1]).max() <= 3e-4
    P = np.sort(ref["prob"], axis=0)
    sure = (P[-1] - P[-2]) > 1e-3
    assert np.array_equal(lab[sure], ref["labels"][sure])
    # the two solvers agree to the solver tolerance, with the same iteration counts (+-3)
    assert np.abs(outs["streaming"]["prob"] - prob).max() <= 2e-5
    it_r = outs["resident"]["iters"].astype(int)
    it_s = outs["streaming"]["iters"].astype(int)
    assert np.abs(it_r - it_s).max() <= 3, (it_r, it_s)


def test_resident_multi_rhs_bitwise_and_linearity():
    """nrhs = 2 on 64^3 bricks: each (rhs, brick) pair equals its own single-rhs resident solve
    bit for bit; values' = 1 - values gives x' = 1 - x (linearity of L_UU x_U = -B^T x_S)
    to the solver tolerance."""
    p = wl.cfg2(bricks=[3, 77, 200])
    two = wl.Problem("two", p.vol, p.dtype, p.fixed,
                     np.concatenate([p.values, (1.0 - p.values).astype(np.float32)]),
                     p.beta, p.eps, p.tol, p.max_iter, p.tol_mode, p.scale, p.offset)
    o = resident(two)
    assert o["prob"].shape[0] == 2
    for r in range(2):
        one = wl.Problem("one", p.vol, p.dtype, p.fixed, two.values[r:r + 1].copy(), p.beta,
                         p.eps, p.tol, p.max_iter, p.tol_mode, p.scale, p.offset)
        s = resident(one)
        assert np.array_equal(s["prob"][0], o["prob"][r])
        assert np.array_equal(s["iters"][0], o["iters"][r])
        assert np.array_equal(s["resid"][0], o["resid"][r])
        if r == 0:
            assert np.array_equal(s["labels"], o["labels"])   # labels = prob[0] > 0.5
    assert np.abs(o["prob"][0] + o["prob"][1] - 1.0).max() <= 2e-5


def test_l2_workers_bitwise_batch_invariant():
    """RW_OPT_L2_WORKERS (default on): 4-CTA worker clusters on the SMs the 64^3 16-CTA
    clusters leave free reproduce the resident arithmetic from global memory, so the whole
    batch is bit-identical with and without them, whichever cluster solved a brick."""
    p = wl.cfg2(bricks=list(range(0, 512, 4)))          # 128 bricks: workers take some
    on = resident(p)
    with rwb.l2_workers(False):
        off = resident(p)
    for k in ("prob", "iters", "resid", "status", "labels"):
        assert np.array_equal(on[k], off[k]), k
    alone = resident(p.subset([77]))
    assert np.array_equal(alone["prob"][0, 0], on["prob"][0, 77])
