"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot solve a 67M-unknown system in test time, so full-size checks are
(a) oracle solves of sampled bricks of the full 512-brick batch, and (b) properties that hold
at any size and pin the answer: the fp64 residual of the GPU solution of the *plain*
definition L_UU x_U = -B^T x_S computed matrix-free from the oracle's fp64 weight
planes, the maximum principle, Sigma_k p_k = 1 for the multi-label solve (linearity), the
argmax rule, and the bit-exact 2^3-mean pyramid on aligned sub-cubes.
"""
import numpy as np
import pytest
import torch

import paper_2103_09564_b200 as rwb
import workloads as wl
from oracle import rw_oracle as ro
from oracle import pyramid_oracle as po
from gpu_helpers import dev, assert_prob_parity, assert_label_parity

pytestmark = pytest.mark.gpu


def residual_fp64(g, fixed, values, x, beta, eps):
    """||b - L_UU x_U|| / ||b|| for one brick, matrix-free in fp64 from the oracle's weight
    planes: (L x)_i = sum_j w_ij (x_i - x_j) over unknown i (x_S = values on S)."""
    W = ro.weight_planes(g, beta, eps)
    fx = fixed.astype(bool)
    xs = np.where(fx, values, x).astype(np.float64)
    Lx = np.zeros_like(xs)
    bvec = np.zeros_like(xs)
    xsS = np.where(fx, values, 0.0)
    for ax in range(3):
        sl_p = [slice(None)] * 3
        sl_q = [slice(None)] * 3
        sl_p[2 - ax] = slice(0, -1)      # W[0] is the x (last) axis, W[2] the z axis
        sl_q[2 - ax] = slice(1, None)
        sp, sq = tuple(sl_p), tuple(sl_q)
        w = W[ax][sp]
        d = xs[sp] - xs[sq]
        Lx[sp] += w * d           # edge contributes w (x_p - x_q) to p ...
        Lx[sq] -= w * d           # ... and w (x_q - x_p) to q
        bvec[sp] += w * xsS[sq]
        bvec[sq] += w * xsS[sp]
    # row i of L x with all x (fixed included) = (L_UU x_U)_i - (B^T x_S)_i -> residual
    r = np.where(fx, 0.0, -Lx)
    bU = np.where(fx, 0.0, bvec)
    return np.linalg.norm(r) / np.linalg.norm(bU)


def local_parity(g, fixed, values, x, beta, eps, z0, y0, x0, m):
    """Oracle check of a full-size solution inside an m^3 sub-block: the fp64 oracle solves
    the sub-block with the seeds inside and the GPU solution on its one-voxel outer shell as
    Dirichlet data (the discrete equations of P:77 restricted to the block); the interior must
    match the GPU solution.  Returns max |dp| over the interior."""
    sl = (slice(z0, z0 + m), slice(y0, y0 + m), slice(x0, x0 + m))
    shell = np.ones((m, m, m), bool)
    shell[1:-1, 1:-1, 1:-1] = False
    fx = fixed[sl].astype(bool) | shell
    vals = np.where(fixed[sl].astype(bool), values[sl], x[sl]).astype(np.float64)
    o = ro.solve_brick(g[sl], fx, vals, beta, eps, tol=1e-11)
    ref = np.where(fx, vals, np.clip(o["x"], 0, 1))
    return float(np.abs(ref - x[sl])[1:-1, 1:-1, 1:-1].max())


def _oracle_brick(sub):
    """One cfg2 brick through the fp64 oracle (run in a worker process, one core each: the
    BLAS dots of 16 workers would otherwise each try to use every core)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        return ro.solve_problem(sub, tol=1e-10)["prob"]


def test_cfg2_full_batch_in_bench_configuration():
    """The whole 512 x 64^3 batch through the default (auto -> resident) solver exactly as
    bench.py runs it.  34 bricks element by element against the fp64 oracle: the bricks
    with the most and the fewest iterations plus 32 spread over the batch; every brick by
    the fp64 residual of the plain definition."""
    import concurrent.futures as cf
    import multiprocessing as mp
    import os
    p = wl.cfg2(batch=512, workers=8)
    out = rwb.solve_bricks(dev(p.fixed), dev(p.values), vol=dev(p.vol), beta=p.beta, eps=p.eps,
                           tol=p.tol, max_iter=p.max_iter, labels=True)
    torch.cuda.synchronize()
    prob = out["prob"].cpu().numpy()
    st = out["status"].cpu().numpy()
    it = out["iters"].cpu().numpy()
    assert (st == 1).all() and it.min() > 100 and it.max() < p.max_iter
    assert prob.min() >= 0.0 and prob.max() <= 1.0
    labels = out["labels"].cpu().numpy()
    ids = sorted({int(np.argmax(it[0])), int(np.argmin(it[0]))} | set(range(0, 512, 16)))
    assert len(ids) >= 32
    with cf.ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 1),
                                mp_context=mp.get_context("spawn")) as ex:
        refs = list(ex.map(_oracle_brick, [p.subset([b]) for b in ids]))
    for b, ref in zip(ids, refs):
        assert_prob_parity(prob[:, b:b + 1], ref)
        assert_label_parity(labels[b], ref[0, 0])
    for b in range(3, 512, 8):
        g = ro.normalise(p.vol[b], p.scale, p.offset)
        rel = residual_fp64(g, p.fixed[b], p.values[0, b], prob[0, b], p.beta, p.eps)
        assert rel <= 2e-5, (b, rel)       # fp32 iterate at rel. tol 1e-6


def test_cfg3_full_size_residual_and_maximum_principle():
    """512x512x256 int16 CT phantom (one 67M-voxel system, streaming passes)."""
    p = wl.cfg3()
    out = rwb.solve_bricks(dev(p.fixed), dev(p.values), vol=dev(p.vol), beta=p.beta, eps=p.eps,
                           tol=p.tol, max_iter=p.max_iter, norm=(p.scale, p.offset))
    torch.cuda.synchronize()
    assert int(out["status"][0, 0]) == 1 and float(out["resid"][0, 0]) <= 1e-6
    x = out["prob"].cpu().numpy()[0, 0]
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    # fp32 floor: x = x0 + sum alpha p accumulated in fp32 over ~3 000 iterations carries
    # ~1e-6 rounding noise per voxel, which the true residual amplifies (R5c)
    rel = residual_fp64(g, p.fixed[0], p.values[0, 0], x, p.beta, p.eps)
    assert rel <= 1e-3, rel
    assert x.min() >= 0.0 and x.max() <= 1.0
    # five fixed sub-blocks (two in opposite volume corners) + seven seeded random ones
    rng = np.random.default_rng(31)
    blocks = [(100, 200, 200), (40, 300, 120), (200, 60, 400), (0, 0, 0), (232, 488, 488)]
    blocks += [(int(rng.integers(0, 233)), int(rng.integers(0, 489)), int(rng.integers(0, 489)))
               for _ in range(7)]
    for (z0, y0, x0) in blocks:
        d = local_parity(g, p.fixed[0], p.values[0, 0], x, p.beta, p.eps, z0, y0, x0, 24)
        assert d <= 1e-4, ((z0, y0, x0), d)


def test_cfg4_full_size_multilabel_properties():
    """256^3, K = 4, three RHS on one operator: Sigma p <= 1 (class 4 = 1 - Sigma, linearity),
    seeds keep their class, labels are the argmax (ties to the lowest id), fp64 residual of
    every solved class."""
    lp = wl.cfg4()
    out = rwb.solve_labels(dev(lp.labels), lp.K, vol=dev(lp.vol), beta=lp.beta, eps=lp.eps,
                           tol=lp.tol, max_iter=lp.max_iter)
    torch.cuda.synchronize()
    prob = out["prob"].cpu().numpy()[:, 0]
    lab = out["labels"].cpu().numpy()[0]
    seeds = lp.labels[0]
    s = prob.astype(np.float64).sum(0)
    assert s.max() <= 1.0 + 1e-4
    assert np.array_equal(lab[seeds > 0], seeds[seeds > 0])
    allp = np.concatenate([prob, np.clip(1.0 - prob.sum(0, keepdims=True), 0, 1)], 0)
    want = np.argmax(allp, axis=0) + 1
    assert np.mean(want == lab) > 0.9999     # fp32 sums of ties may differ in rare voxels
    g = ro.normalise(lp.vol[0], lp.scale, lp.offset)
    fixed = seeds > 0
    for k in range(lp.K - 1):
        vk = (seeds == k + 1).astype(np.float64)
        rel = residual_fp64(g, fixed, vk, prob[k], lp.beta, lp.eps)
        assert rel <= 1e-3, (k, rel)          # fp32 floor, see the cfg3 test
    # element-wise: every solved class and the derived class K = 1 - sum (R11) inside 24^3
    # sub-blocks that straddle class boundaries, solved by the oracle with the GPU solution
    # on their shell (the discrete equations of P:77 restricted to the block)
    pK = np.clip(1.0 - prob.astype(np.float64).sum(0), 0.0, 1.0)
    fields = [prob[k].astype(np.float64) for k in range(lp.K - 1)] + [pK]
    for k, xk in enumerate(fields):
        vk = (seeds == k + 1).astype(np.float64)
        for (z0, y0, x0) in [(100, 110, 90), (60, 128, 150), (150, 40, 120), (0, 0, 0),
                             (232, 232, 232), (20, 200, 60)]:
            d = local_parity(g, fixed, vk, xk, lp.beta, lp.eps, z0, y0, x0, 24)
            assert d <= 1e-4, (k, (z0, y0, x0), d)


def test_pyramid_2048_aligned_subcubes_bit_exact():
    """Config 5's 2048^3 u16 volume size -> 5 levels; two aligned 256^3 sub-cubes (one at
    each corner) against the integer oracle: the 2^3 mean is local, so a sub-cube's pyramid
    is the matching region of the full one."""
    d = 2048
    gen = torch.Generator(device="cuda").manual_seed(11)
    vol = torch.randint(0, 65536, (d, d, d), dtype=torch.int32, device="cuda",
                        generator=gen).to(torch.uint16)
    outs = rwb.build_pyramid(vol, 5)
    torch.cuda.synchronize()
    for o in (0, d - 256):
        sub = vol[o:o + 256, o:o + 256, o:o + 256].cpu().numpy()
        ref = po.pyramid(sub, 5)
        for l, (g, r) in enumerate(zip(outs, ref)):
            k = o >> (l + 1)
            e = 256 >> (l + 1)
            assert np.array_equal(g[k:k + e, k:k + e, k:k + e].cpu().numpy(), r), (o, l)
