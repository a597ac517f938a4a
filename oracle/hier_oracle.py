"""fp64 oracle of the hierarchical random walker driver (TEST INFRASTRUCTURE; see
oracle/__init__.py).  SURVEY.md §8(f) row f1.

Citations: P:n = /root/reference/PAPER.md line n (§IV); S:n = SPEC.md line n
(readings only); readings R22-R28 are restated in DESIGN.md §3.

The procedure, level by level from the root (coarsest LOD level) down to the full
resolution, written in the paper's order:

  levels    volume D^3 with D = s 2^k: level l has D/2^l voxels per axis, l = k is the root
            (one brick); intensities per level = the integer 2^3-mean pyramid (P:71,
            pyramid_oracle).
  seeds     full-resolution label volume: 0 unseeded, 1 foreground, 2 background (the
            rasterised T_n(l), reading R22).  At level l a voxel carries the labels of
            the full-resolution voxels it covers; foreground and background together is a
            conflict cfl: the voxel is left unseeded.
  root      Eq. 1: x = rw(n_0, T(l)) on the whole root level, x0 = 0.5.
  level l   for every active brick n (s^3 at level l): the expanded window N(n) of side
            s_e = floor(e s) (Eq. 3) with margin ceil((s_e - s)/2) on the low side,
            shifted inward to stay inside the level (reading R23); seeds L(N(n), l) = the
            user seeds in the window  U  continuous seeds on the window's faces that are
            interior to the volume, sampled from the parent level's probability field
            (sample_border; reading R24; user seeds win); initial guess = the
            parent field sampled at every window voxel (reading R25); solve; contract
            N^-1: the central s^3 goes to the level's probability field.
  parent    field sampling = trilinear interpolation at the child voxel centre (i + 0.5)/2 - 0.5
            in parent voxel units, clamped at the level border (reading R25).
  pruning   P:139-161: prunable(n) = (hom(n) or dt(n)) and not cfl(n) with hom = max - min <
            t_hom, dt = min - 0.5 > t_bin or 0.5 - max > t_bin over the brick's s^3
            probabilities, cfl = a conflict voxel inside the brick at its level.  Children of
            prunable bricks are not solved; every level's field starts as the trilinear
            upsample of the parent field and solved bricks overwrite their s^3, so sampling
            a pruned region falls back to the nearest solved ancestor (reading R26).
  dims      volumes need not be cubic nor s 2^k ("bricks at the border of the
            volume may be smaller than s^3 voxels"; reading R31): level l+1 has dims
            ceil(d_l / 2) per axis (the pyramid's); the root is the first level whose
            dims are all <= s; a level has ceil(d_l / s) bricks per axis, the last one per
            axis smaller; brick B's children are the bricks 2B + (0|1) that exist; a window
            has side min(s_e, d_l) per axis (a level narrower than s_e is taken whole).
Solves use rw_oracle.solve_brick (fp64 Jacobi-PCG); the output is the level-0 field.
"""
from __future__ import annotations

import math

import numpy as np

from . import pyramid_oracle
from . import rw_oracle as ro


def seed_bits(seeds):
    """Full-resolution labels -> bits (1 = foreground, 2 = background)."""
    s = np.asarray(seeds)
    return ((s == 1).astype(np.uint8) | ((s == 2).astype(np.uint8) << 1))


def seed_bit_pyramid(seeds, levels):
    """Level l bits = OR of the bits of the (up to 2^3) present children at level l-1
    (reading R22); dims ceil(d/2) per axis (R31); level 0 first."""
    out = [seed_bits(seeds)]
    for _ in range(levels - 1):
        b = out[-1]
        nz, ny, nx = b.shape
        oz, oy, ox = (nz + 1) // 2, (ny + 1) // 2, (nx + 1) // 2
        pad = np.zeros((2 * oz, 2 * oy, 2 * ox), np.uint8)     # absent children: no label
        pad[:nz, :ny, :nx] = b
        c = pad.reshape(oz, 2, oy, 2, ox, 2)
        out.append(np.bitwise_or.reduce(np.bitwise_or.reduce(np.bitwise_or.reduce(c, 5), 3), 1))
    return out


def level_dims(shape, s):
    """Per-level dims (level 0 first) down to the root, the first level with every dim <= s
    (reading R31)."""
    dims = [tuple(int(a) for a in shape)]
    while max(dims[-1]) > s:
        dims.append(tuple((a + 1) // 2 for a in dims[-1]))
    return dims


def seeds_from_bits(bits):
    """(fixed, value): a voxel is seeded iff exactly one of fg / bg is present."""
    fg = (bits & 1) > 0
    bg = (bits & 2) > 0
    fixed = fg ^ bg
    return fixed, np.where(fg & ~bg, 1.0, 0.0)


def parent_coord(i):
    """Parent-voxel coordinate of child voxel centre i (reading R25)."""
    return (np.asarray(i, np.float64) + 0.5) / 2.0 - 0.5


def sample_parent(P, zs, ys, xs):
    """Trilinear sample of the parent field P at the parent coordinates of child voxel
    indices (zs, ys, xs) (1-D index arrays per axis, outer product), clamped at the border."""
    out = np.zeros((len(zs), len(ys), len(xs)))
    idx, wts = [], []
    for n, c in zip(P.shape, (zs, ys, xs)):
        u = np.clip(parent_coord(c), 0.0, n - 1)
        i0 = np.floor(u).astype(int)
        i1 = np.minimum(i0 + 1, n - 1)
        f = u - i0
        idx.append((i0, i1))
        wts.append((1.0 - f, f))
    for a in range(2):
        for b in range(2):
            for c in range(2):
                w = (wts[0][a][:, None, None] * wts[1][b][None, :, None] * wts[2][c][None, None, :])
                out += w * P[np.ix_(idx[0][a], idx[1][b], idx[2][c])]
    return out


def upsample(P, shape):
    """Dense trilinear upsample of the parent field onto a level of `shape`."""
    return sample_parent(P, np.arange(shape[0]), np.arange(shape[1]), np.arange(shape[2]))


def window_origin(brick, s, se, D):
    """Reading R23: low margin ceil((se - s)/2), shifted inward to fit [0, D); a level
    narrower than se is taken whole (R31)."""
    side = min(se, D)
    o = brick * s - int(math.ceil((se - s) / 2))
    return int(min(max(o, 0), D - side))


def window_system(P_par, fx_l, val_l, brick, s, se, Dl):
    """The Dirichlet data of one expanded window N(n) at level l (Eq. 3).

    Returns (w0, fixed, values, samp): the window origin (reading R23), the fixed mask and
    values = the user seeds inside the window plus the continuous border seeds of
    sample_border (reading R24): every voxel of the window's one-voxel shell on a face
    interior to the volume (w0 > 0 for the low face, w0 + se < Dl for the high face) that is
    not a user seed takes the parent field sampled at its centre (reading R25); faces on
    the volume boundary stay Neumann (reading c4).  samp = the parent field sampled at every
    window voxel (the initial guess)."""
    Dl = (Dl,) * 3 if np.isscalar(Dl) else tuple(Dl)
    w0 = [window_origin(c, s, se, d) for c, d in zip(brick, Dl)]
    side = [min(se, d) for d in Dl]
    sl = tuple(slice(a, a + w) for a, w in zip(w0, side))
    zs, ys, xs = (np.arange(a, a + w) for a, w in zip(w0, side))
    samp = sample_parent(P_par, zs, ys, xs)
    fixed = fx_l[sl].copy()
    values = np.where(fixed, val_l[sl], 0.0)
    shell = np.zeros(tuple(side), bool)
    for ax in range(3):
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[ax] = 0
        hi[ax] = side[ax] - 1
        if w0[ax] > 0:
            shell[tuple(lo)] = True
        if w0[ax] + side[ax] < Dl[ax]:
            shell[tuple(hi)] = True
    border = shell & ~fixed
    values = np.where(border, samp, values)
    return w0, fixed | border, values, samp


def hier_segment(vol, seeds, s=32, e=1.25, t_hom=0.3, t_bin=0.01, beta=100.0, eps=1e-6,
                 tol=1e-10, max_iter=100000, scale=1.0 / 65535, offset=0.0, prune=True,
                 prev=None, t_inc=0.01):
    """Oracle of rw_hier_segment / rw_hier_segment_ooc.  vol/seeds [nz, ny, nx] (z, y, x), any
    dims (reading R31); the in-HBM driver takes cubic D = s 2^k.

    prev: the dict a previous call returned (same volume and geometry) -> incremental
    labelling H_it (reading R27): every solved brick whose previous node was
    computed, whose new solution differs from the previous one by less than t_inc
    everywhere in its s^3 and that has no seed conflict involving a changed label
    keeps its previous values and its whole previous subtree; recomputed bricks start from
    their previous solution.

    Returns dict(prob [D,D,D] fp64 in [0,1], stats per level, fields [level] (level 0
    first), computed [level] = set of bricks holding a computed node, bits [level]).
    """
    vol = np.asarray(vol)
    dims = level_dims(vol.shape, s)          # reading R31; cubic s 2^k: D / 2^l
    k = len(dims) - 1
    levels = k + 1
    se = int(math.floor(e * s))
    inc = prev is not None
    vols = [vol] + (pyramid_oracle.pyramid(vol, k) if k > 0 else [])
    bits = seed_bit_pyramid(seeds, levels)
    stats = [dict(active=0, solved=0, pruned_hom=0, pruned_dt=0, conflict=0, reused=0, iters=0)
             for _ in range(levels)]
    fields = [None] * levels
    computed = [set() for _ in range(levels)]

    def region(b, l):
        return tuple(slice(c * s, min((c + 1) * s, d)) for c, d in zip(b, dims[l]))

    def decide(l, b, xb, old):
        """(state, values kept): reuse (R27) before the pruning rule."""
        if inc and b in prev["computed"][l]:
            cb, ob = bits[l][region(b, l)], prev["bits"][l][region(b, l)]
            dconf = np.any((cb == 3) & (cb != ob))
            if not dconf and np.max(np.abs(xb - old)) < t_inc:
                return "reused", old
        return _prune_state(b, xb, bits[l][region(b, l)], t_hom, t_bin, prune), xb

    # ---- root (Eq. 1)
    g = ro.normalise(vols[k], scale, offset)
    fixed, val = seeds_from_bits(bits[k])
    o = ro.solve_brick(g, fixed, val, beta, eps, tol, max_iter,
                       x0=prev["fields"][k] if inc else None)
    xr = np.where(fixed, val, np.clip(o["x"], 0.0, 1.0))
    st, kept = decide(k, (0, 0, 0), xr, prev["fields"][k] if inc else None)
    fields[k] = kept.copy()
    computed[k].add((0, 0, 0))
    stats[k].update(active=1, solved=1, iters=o["iters"])
    _count(stats[k], st)
    state = {(0, 0, 0): st}            # per brick of the previous (coarser) level
    reused_desc = set()                # bricks under a reused node

    # ---- levels k-1 .. 0 (Eq. 3 with H_p and H_it)
    for l in range(k - 1, -1, -1):
        Dl = dims[l]
        nb = tuple((d + s - 1) // s for d in Dl)

        def kids(b):
            return {(2 * b[0] + cz, 2 * b[1] + cy, 2 * b[2] + cx)
                    for cz in range(2) for cy in range(2) for cx in range(2)
                    if 2 * b[0] + cz < nb[0] and 2 * b[1] + cy < nb[1] and 2 * b[2] + cx < nb[2]}
        active, keep = set(), set()
        for b, stt in state.items():
            if stt in (None, "cfl"):
                active |= kids(b)
            elif stt == "reused":
                keep |= kids(b)
        for b in reused_desc:
            keep |= kids(b)
        P_par = fields[l + 1]
        up = upsample(P_par, Dl)
        F = prev["fields"][l].copy() if inc else up.copy()
        for b in ((bz, by, bx) for bz in range(nb[0]) for by in range(nb[1]) for bx in range(nb[2])):
            if b not in active and b not in keep:
                F[region(b, l)] = up[region(b, l)]     # pruned region: nearest solved ancestor
        computed[l] = {b for b in keep if inc and b in prev["computed"][l]}
        gl = ro.normalise(vols[l], scale, offset)
        fx_l, val_l = seeds_from_bits(bits[l])
        stats[l]["active"] = len(active)
        new_state = {}
        for (bz, by, bx) in sorted(active):
            w0, fixed, values, samp = window_system(P_par, fx_l, val_l, (bz, by, bx), s, se, Dl)
            sl = tuple(slice(a, a + w) for a, w in zip(w0, fixed.shape))
            x0 = prev["fields"][l][sl] if inc else samp
            o = ro.solve_brick(gl[sl], fixed, values, beta, eps, tol, max_iter, x0=x0)
            xw = np.where(fixed, values, np.clip(o["x"], 0.0, 1.0))
            # contract: the brick's own s^3 (smaller at the volume border)
            rg = region((bz, by, bx), l)
            xb = xw[tuple(slice(r.start - a, r.stop - a) for r, a in zip(rg, w0))]
            old = prev["fields"][l][rg] if inc else None
            stt, kept = decide(l, (bz, by, bx), xb, old)
            F[rg] = kept
            computed[l].add((bz, by, bx))
            stats[l]["solved"] += 1
            stats[l]["iters"] += o["iters"]
            new_state[(bz, by, bx)] = stt
            _count(stats[l], stt)
        fields[l] = F
        reused_desc = keep
        state = new_state
    return dict(prob=fields[0], stats=stats, fields=fields, computed=computed, bits=bits)


def _prune_state(b, xb, cb, t_hom, t_bin, prune):
    """None (keep refining: children are solved) or 'hom' / 'dt'; a seed
    conflict inside the brick (bits cb of its region) vetoes pruning ('cfl')."""
    if not prune or np.any(cb == 3):
        return "cfl" if np.any(cb == 3) else None
    mn, mx = float(xb.min()), float(xb.max())
    if t_hom >= 0 and mx - mn < t_hom:
        return "hom"
    if t_bin >= 0 and (mn - 0.5 > t_bin or 0.5 - mx > t_bin):
        return "dt"
    return None


def _count(stat, st):
    if st == "hom":
        stat["pruned_hom"] += 1
    elif st == "dt":
        stat["pruned_dt"] += 1
    elif st == "cfl":
        stat["conflict"] += 1
    elif st == "reused":
        stat["reused"] += 1


def hier_segment_labels(vol, labels, K, s=32, e=1.25, t_hom=0.3, prune=True, prev=None, **kw):
    """Multi-class hierarchical segmentation ("run once for each class, where only
    seeds for the current class are considered foreground and all other seeds as
    background ... the class of a voxel is the one that maximizes the foreground
    probability"; only homogeneity pruning, dt disabled).  `labels`:
    0 unseeded, 1..K class seeds.  `prev`: an earlier result on the same volume -> each class
    runs H_it from its own previous run.  Returns dict(labels [D,D,D] in 1..K with
    ties to the lowest class id (reading R11), prob [K][D,D,D], stats [K], runs [K])."""
    labels = np.asarray(labels)
    P, S, R = [], [], []
    for k in range(1, K + 1):
        seeds = np.where(labels == k, 1, np.where(labels > 0, 2, 0)).astype(np.uint8)
        o = hier_segment(vol, seeds, s=s, e=e, t_hom=t_hom, t_bin=-1.0, prune=prune,
                         prev=None if prev is None else prev["runs"][k - 1], **kw)
        P.append(o["prob"])
        S.append(o["stats"])
        R.append(o)
    P = np.asarray(P)
    return dict(labels=(np.argmax(P, axis=0) + 1).astype(np.uint8), prob=P, stats=S, runs=R)
