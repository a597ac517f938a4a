"""fp64 oracle of the paper's alternative edge-weight functions (TEST INFRASTRUCTURE; see
oracle/__init__.py).  SURVEY.md §8(f) row f3.

Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n (readings only);
readings R19-R21 are restated in DESIGN.md §3.

  poisson   ([61], used in the paper's case study):
              w_pq = exp(-1/2 (sqrt(n[p]) - sqrt(n[q]))^2) + eps
            n = raw voxel value * count_scale, clipped at 0 (reading R19: the formula has no
            beta, so n is the photon count, not the [0,1]-normalised intensity).
  gaussian  ([28] "derived from the first estimated ... global variance sigma^2 of
            pixel intensity differences"; reading R20 after S:235):
              sigma^2 = mean over the brick's 6-neighbour edges of (g_p - g_q)^2, floored
                        at 1e-8;   w_pq = exp(-(g_p - g_q)^2 / (2 sigma^2)) + eps
  ttest     (Bian et al. [29]: "the P-value of the H_0 hypothesis that the pixel
            distributions defined by values sampled around p and q have the same mean";
            reading R21 after S:234):
              samples = g over the (2R+1)^3 neighbourhood of p (resp. q), clipped at the
              brick border; Welch's statistic t = (m_p - m_q) / sqrt(v_p/n_p + v_q/n_q)
              with unbiased sample variances floored at 1e-8; two-tailed p-value under the
              normal approximation, P = erfc(|t| / sqrt 2);  w_pq = P + eps.
Every weight gets the additive floor eps of reading c1/R1, like the Grady weight.

The layout is that of rw_brick_weights: W[a][z,y,x] = w(voxel, voxel + e_a), 0 where the
neighbour is outside the brick.  Plain numpy; no blocking or fusion.
"""
from __future__ import annotations

import math

import numpy as np

SIGMA2_FLOOR = 1e-8
VAR_FLOOR = 1e-8

KINDS = {"grady": 0, "poisson": 1, "gaussian": 2, "ttest": 3}


def _forward_pairs(a):
    """(a_p, a_q) views for the three axes with q = p + e_a (x, y, z)."""
    return ((a[:, :, :-1], a[:, :, 1:]), (a[:, :-1, :], a[:, 1:, :]), (a[:-1, :, :], a[1:, :, :]))


def _planes(fn, *arrays):
    """W[3] planes from an edge function fn(p-values..., q-values...)."""
    shp = arrays[0].shape
    W = np.zeros((3,) + shp)
    sl = ((slice(None), slice(None), slice(0, -1)), (slice(None), slice(0, -1), slice(None)),
          (slice(0, -1), slice(None), slice(None)))
    for ax in range(3):
        pairs = [_forward_pairs(a)[ax] for a in arrays]
        W[ax][sl[ax]] = fn(*[p for p, _ in pairs], *[q for _, q in pairs])
    return W


def poisson_counts(vol, count_scale=1.0):
    """Reading R19: n = raw value * count_scale, clipped at 0 (counts are non-negative)."""
    return np.clip(np.asarray(vol, np.float64) * float(count_scale), 0.0, None)


def poisson_planes(counts, eps):
    """w = exp(-1/2 (sqrt(n_p) - sqrt(n_q))^2) + eps."""
    s = np.sqrt(np.asarray(counts, np.float64))
    return _planes(lambda sp, sq: np.exp(-0.5 * (sp - sq) ** 2) + eps, s)


def gaussian_sigma2(g):
    """Reading R20: mean of (g_p - g_q)^2 over all 6-neighbour edges of the brick, floored."""
    g = np.asarray(g, np.float64)
    tot, cnt = 0.0, 0
    for gp, gq in _forward_pairs(g):
        tot += float(np.sum((gq - gp) ** 2))
        cnt += gp.size
    return max(tot / cnt, SIGMA2_FLOOR) if cnt else SIGMA2_FLOOR


def gaussian_planes(g, eps):
    """P:127 / [28]: w = exp(-(g_p - g_q)^2 / (2 sigma^2)) + eps, sigma^2 per brick."""
    g = np.asarray(g, np.float64)
    s2 = gaussian_sigma2(g)
    return _planes(lambda gp, gq: np.exp(-((gp - gq) ** 2) / (2.0 * s2)) + eps, g)


def ttest_stats(g, radius=1):
    """Per voxel: (n, mean, unbiased variance floored) of the (2R+1)^3 neighbourhood
    clipped at the brick border (reading R21).  Loops over the neighbourhood offsets."""
    g = np.asarray(g, np.float64)
    nz, ny, nx = g.shape
    R = int(radius)
    S = np.zeros_like(g)
    N = np.zeros_like(g)
    for dz in range(-R, R + 1):
        for dy in range(-R, R + 1):
            for dx in range(-R, R + 1):
                src = g[max(dz, 0):nz + min(dz, 0), max(dy, 0):ny + min(dy, 0),
                        max(dx, 0):nx + min(dx, 0)]
                dst = (slice(max(-dz, 0), nz + min(-dz, 0)), slice(max(-dy, 0), ny + min(-dy, 0)),
                       slice(max(-dx, 0), nx + min(-dx, 0)))
                S[dst] += src
                N[dst] += 1
    M = S / N
    SS = np.zeros_like(g)
    for dz in range(-R, R + 1):
        for dy in range(-R, R + 1):
            for dx in range(-R, R + 1):
                src = g[max(dz, 0):nz + min(dz, 0), max(dy, 0):ny + min(dy, 0),
                        max(dx, 0):nx + min(dx, 0)]
                dst = (slice(max(-dz, 0), nz + min(-dz, 0)), slice(max(-dy, 0), ny + min(-dy, 0)),
                       slice(max(-dx, 0), nx + min(-dx, 0)))
                SS[dst] += (src - M[dst]) ** 2
    V = np.where(N > 1, SS / np.maximum(N - 1, 1), 0.0)
    return N, M, np.maximum(V, VAR_FLOOR)


def welch_t(mp, vp, np_, mq, vq, nq):
    """Welch's two-sample statistic (reading R21)."""
    return (mp - mq) / np.sqrt(vp / np_ + vq / nq)


def pvalue_normal(t):
    """Two-tailed p-value of t under the normal approximation: erfc(|t| / sqrt 2)."""
    return np.vectorize(lambda x: math.erfc(abs(x) / math.sqrt(2.0)))(t)


def ttest_planes(g, eps, radius=1):
    """P:123-125 / [29]: w_pq = P-value(H_0: same mean around p and q) + eps."""
    N, M, V = ttest_stats(g, radius)
    return _planes(lambda np_, mp, vp, nq, mq, vq:
                   pvalue_normal(welch_t(mp, vp, np_, mq, vq, nq)) + eps, N, M, V)


def planes(kind, vol, scale, offset, eps, beta=100.0, count_scale=1.0, radius=1):
    """Weight planes of one brick for any kind (grady via rw_oracle.weight_planes)."""
    from .rw_oracle import normalise, weight_planes
    if kind == "poisson":
        return poisson_planes(poisson_counts(vol, count_scale), eps)
    g = normalise(vol, scale, offset)
    if kind == "grady":
        return weight_planes(g, beta, eps)
    if kind == "gaussian":
        return gaussian_planes(g, eps)
    if kind == "ttest":
        return ttest_planes(g, eps, radius)
    raise ValueError(kind)


def planes_to_edges(W):
    """Weight planes -> the undirected edge list (i, j, w) rw_oracle.solve_brick consumes."""
    _, nz, ny, nx = W.shape
    idx = np.arange(nz * ny * nx).reshape(nz, ny, nx)
    I, J, Wt = [], [], []
    for ax, (sp, sq) in enumerate(_forward_pairs(idx)):
        I.append(sp.ravel())
        J.append(sq.ravel())
        Wt.append(W[ax][tuple(slice(0, s) for s in sp.shape)].ravel())
    return np.concatenate(I), np.concatenate(J), np.concatenate(Wt)
