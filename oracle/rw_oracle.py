"""Plain fp64 random walker oracle (TEST INFRASTRUCTURE; see oracle/__init__.py).

Citations: ``P:n`` = /root/reference/PAPER.md line n (§III-B "Random Walker Volume
Segmentation"; §V solver settings); ``BJ`` = BASELINE.json north_star;
readings c1..c17 = SURVEY.md §8(c), restated in DESIGN.md §3.

What it computes (per brick b and right-hand side r):
  g      = clamp(v*scale + offset, 0, 1)                              (reading c2)
  w_pq   = exp(-beta (g_p - g_q)^2) + eps for every 6-neighbour edge    (P:77 + BJ, c1)
  L      = weighted graph Laplacian of the brick graph (no edges leave the brick, c4)
  split x into x_S (fixed: seeds + Dirichlet faces) and x_U; solve
           L_UU x_U = -B^T x_S  =: b,   b_i = sum_{j in S, j~i} w_ij x_j
  by Jacobi-preconditioned CG (P:197, P:33 fn 2) to ||r||_2 <= tol ||b||_2 on the
  recurrence residual (reading c5), then clamp to [0,1] (c9).
Multi-class: one one-vs-rest solve per class, class = argmax, ties -> lowest id.

Every step is the textbook definition: edges enumerated per axis, the sparse matrix is
assembled entry by entry (scipy COO -> CSR is only the container), CG is the
Hestenes-Stiefel recurrence written out.  No blocking, fusion or reordering.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# ----------------------------------------------------------------------------- weights

def normalise(vol, scale, offset):
    """Reading c2: intensity -> [0,1] as g = clamp(v*scale + offset, 0, 1), fp64."""
    return np.clip(np.asarray(vol, np.float64) * float(scale) + float(offset), 0.0, 1.0)


def edge_list(g, beta, eps):
    """All undirected 6-neighbour edges of one brick g[nz, ny, nx] ("edges between
    6-neighbors") with Grady weights w = exp(-beta (g_p - g_q)^2) + eps (c1).

    Returns (i, j, w): flat voxel indices (x fastest) and fp64 weights; i < j, j = i + e_a.
    """
    nz, ny, nx = g.shape
    idx = np.arange(nz * ny * nx).reshape(nz, ny, nx)
    I, J, Wt = [], [], []
    for sl_p, sl_q in (((slice(None), slice(None), slice(0, -1)), (slice(None), slice(None), slice(1, None))),   # x
                       ((slice(None), slice(0, -1), slice(None)), (slice(None), slice(1, None), slice(None))),   # y
                       ((slice(0, -1), slice(None), slice(None)), (slice(1, None), slice(None), slice(None)))):  # z
        gp, gq = g[sl_p], g[sl_q]
        I.append(idx[sl_p].ravel())
        J.append(idx[sl_q].ravel())
        Wt.append((np.exp(-float(beta) * (gp - gq) ** 2) + float(eps)).ravel())
    return np.concatenate(I), np.concatenate(J), np.concatenate(Wt)


def weight_planes(g, beta, eps):
    """The same weights laid out as three planes W_a[z,y,x] = w(voxel, voxel + e_a), with 0
    where voxel + e_a is outside the brick (reading c4) -- the layout of rw_brick_weights."""
    nz, ny, nx = g.shape
    W = np.zeros((3, nz, ny, nx))
    W[0, :, :, :-1] = np.exp(-beta * (g[:, :, 1:] - g[:, :, :-1]) ** 2) + eps
    W[1, :, :-1, :] = np.exp(-beta * (g[:, 1:, :] - g[:, :-1, :]) ** 2) + eps
    W[2, :-1, :, :] = np.exp(-beta * (g[1:, :, :] - g[:-1, :, :]) ** 2) + eps
    return W

# ----------------------------------------------------------------------------- system

class System:
    """L_UU, b and bookkeeping for one brick and one RHS."""

    def __init__(self, n, edges, fixed, xs):
        i, j, w = edges
        fixed = np.asarray(fixed, bool).ravel()
        xs = np.asarray(xs, np.float64).ravel()
        self.n = n
        self.fixed = fixed
        self.U = np.flatnonzero(~fixed)
        self.S = np.flatnonzero(fixed)
        # full Laplacian L = D - A, assembled entry by entry (duplicates summed by COO)
        rows = np.concatenate([i, j, i, j])
        cols = np.concatenate([i, j, j, i])
        vals = np.concatenate([w, w, -w, -w])
        L = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
        self.L_UU = L[self.U][:, self.U].tocsr()
        B_US = L[self.U][:, self.S]             # = -(w_ij) for i in U, j in S
        self.b = -(B_US @ xs[self.S])           # b = -B^T x_S
        self.diag = self.L_UU.diagonal()
        self.xs = xs


def pcg(A, b, x0, dinv, tol, max_iter, tol_mode=0):
    """Jacobi-preconditioned conjugate gradient (P:33 fn 2), Hestenes-Stiefel form.

    Stopping (reading c5): before each iteration, stop if ||r_k||_2 <= tol*||b||_2
    (tol_mode 0) or ||r_k||_2 <= tol (tol_mode 1), r_k the recurrence residual; at most
    max_iter iterations.  Returns (x, iters, ||r||/||b|| or ||r||).
    """
    x = x0.astype(np.float64).copy()
    r = b - A @ x
    z = dinv * r
    p = z.copy()
    rz = r @ z
    bn = np.sqrt(b @ b)
    thresh = tol * bn if tol_mode == 0 else tol
    k = 0
    rn = np.sqrt(r @ r)
    while rn > thresh and k < max_iter:
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        z = dinv * r
        rz_new = r @ z
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
        k += 1
        rn = np.sqrt(r @ r)
    rel = rn / bn if (tol_mode == 0 and bn > 0) else rn
    return x, k, rel


def solve_brick(g, fixed, xs, beta, eps, tol=1e-10, max_iter=100000, x0=None, tol_mode=0,
                edges=None):
    """Random walker solution x (unclamped, full brick) of one brick / one RHS.

    Degenerate cases (ABI contract): no fixed voxel -> x = x0 (default 0.5),
    iters 0; no unknown voxel -> x = x_S; b = 0 -> x_U = 0 exactly (the unique solution).
    Returns dict(x, iters, rel, true_rel).
    """
    shp = g.shape
    n = g.size
    fixed = np.asarray(fixed, bool).ravel()
    xs = np.asarray(xs, np.float64).ravel()
    x0 = (np.full(n, 0.5) if x0 is None else np.asarray(x0, np.float64).ravel())
    if not fixed.any():
        return dict(x=x0.reshape(shp).copy(), iters=0, rel=0.0, true_rel=0.0)
    if fixed.all():
        return dict(x=xs.reshape(shp).copy(), iters=0, rel=0.0, true_rel=0.0)
    if edges is None:
        edges = edge_list(g, beta, eps)
    s = System(n, edges, fixed, xs)
    x = np.where(fixed, xs, x0)
    if not np.any(s.b):
        x[s.U] = 0.0
        return dict(x=x.reshape(shp), iters=0, rel=0.0, true_rel=0.0)
    xu, k, rel = pcg(s.L_UU, s.b, x[s.U], 1.0 / s.diag, tol, max_iter, tol_mode)
    x[s.U] = xu
    tr = np.linalg.norm(s.b - s.L_UU @ xu) / np.linalg.norm(s.b)
    return dict(x=x.reshape(shp), iters=k, rel=rel, true_rel=tr)


def solve_problem(prob, tol=1e-10, max_iter=100000, bricks=None, x0=None, tol_mode=None):
    """Oracle for ``rw_solve_bricks`` on a workloads.Problem.

    Returns dict(x [R,B,nz,ny,nx] unclamped, prob clamped to [0,1] (c9) with fixed voxels
    holding their values, iters [R,B], rel [R,B], true_rel [R,B]).
    ``bricks`` restricts to a subset of batch indices (outputs are then [R, len(bricks)]).
    """
    ids = range(prob.vol.shape[0]) if bricks is None else list(bricks)
    tm = prob.tol_mode if tol_mode is None else tol_mode
    R = prob.values.shape[0]
    xs_out, it, rl, tr = [], [], [], []
    for b in ids:
        g = normalise(prob.vol[b], prob.scale, prob.offset)
        e = edge_list(g, prob.beta, prob.eps)
        xr, ir, rr, tt = [], [], [], []
        for r in range(R):
            o = solve_brick(g, prob.fixed[b], prob.values[r, b], prob.beta, prob.eps, tol,
                            max_iter, None if x0 is None else x0[r, b], tm, edges=e)
            xr.append(o["x"]); ir.append(o["iters"]); rr.append(o["rel"]); tt.append(o["true_rel"])
        xs_out.append(xr); it.append(ir); rl.append(rr); tr.append(tt)
    x = np.transpose(np.asarray(xs_out), (1, 0, 2, 3, 4))
    fixed = prob.fixed[list(ids)].astype(bool)
    vals = prob.values[:, list(ids)].astype(np.float64)
    p = np.where(fixed[None], vals, np.clip(x, 0.0, 1.0))
    return dict(x=x, prob=p, iters=np.asarray(it).T, rel=np.asarray(rl).T,
                true_rel=np.asarray(tr).T)


def threshold(p):
    """P:79 class map by thresholding at 0.5; exactly 0.5 -> background (reading c10)."""
    return (np.asarray(p) > 0.5).astype(np.uint8)


def solve_labels(lp, tol=1e-10, max_iter=100000, bricks=None):
    """Oracle for ``rw_solve_labels``: P:79 / P:107 -- for each class k in 1..K run the
    random walker with seeds of class k as foreground (1) and all other seeds as
    background (0); class = argmax_k x_k with ties to the lowest class id (reading c11).
    All K systems are solved explicitly (the GPU derives class K as 1 - sum).

    Returns dict(prob [K,B,nz,ny,nx] clamped, x unclamped, labels [B,...] in 1..K,
    iters [K,B]).
    """
    ids = range(lp.vol.shape[0]) if bricks is None else list(bricks)
    P, X, IT = [], [], []
    for b in ids:
        g = normalise(lp.vol[b], lp.scale, lp.offset)
        e = edge_list(g, lp.beta, lp.eps)
        lab = lp.labels[b]
        fixed = lab > 0
        pk, xk, ik = [], [], []
        for k in range(1, lp.K + 1):
            xs = (lab == k).astype(np.float64)
            o = solve_brick(g, fixed, xs, lp.beta, lp.eps, tol, max_iter, edges=e)
            xk.append(o["x"])
            pk.append(np.where(fixed, xs.reshape(g.shape), np.clip(o["x"], 0, 1)))
            ik.append(o["iters"])
        P.append(pk); X.append(xk); IT.append(ik)
    P = np.transpose(np.asarray(P), (1, 0, 2, 3, 4))
    X = np.transpose(np.asarray(X), (1, 0, 2, 3, 4))
    labels = (np.argmax(P, axis=0) + 1).astype(np.uint8)   # argmax returns first max
    return dict(prob=P, x=X, labels=labels, iters=np.asarray(IT).T)


# ----------------------------------------------------------------------------- properties
def true_residual(prob, x, b_index=0, r_index=0):
    """||b - L_UU x_U||_2 / ||b||_2 of a given full-brick solution (fp64), for the
    any-size property checks.  ``x`` is [nz, ny, nx]."""
    g = normalise(prob.vol[b_index], prob.scale, prob.offset)
    s = System(g.size, edge_list(g, prob.beta, prob.eps), prob.fixed[b_index],
               prob.values[r_index, b_index])
    xu = np.asarray(x, np.float64).ravel()[s.U]
    bn = np.linalg.norm(s.b)
    return np.linalg.norm(s.b - s.L_UU @ xu) / (bn if bn > 0 else 1.0)
