"""Pins of the hierarchical oracle's continuous border seeds (sample_border, Eq. 2/3) and of
its agreement with the plain random walker on the whole volume.

Citations: P:n = /root/reference/PAPER.md line n.
  P:97  "the solution for the coarser layer serves as an approximation of the *true*
        probability map at the current level (if hypothetically computed on the full volume
        at the current LOD level) and is used to add additional *continuous labels* ... at
        the border of the current brick, i.e., by upsampling from the coarser level".
  P:99  L(n_i, l) = T_{n_i}(l) U sample_border_{n_i}(H(n_{i-1}, l, beta)).
  P:115 s_e = floor(e s); Eq. 3 (expand, solve with border seeds, contract).
Readings R23 (window origin), R24 (which faces carry border seeds), R25 (trilinear sampling
at the child voxel centre) are DESIGN.md §3.

The worked example below is computed by hand (the numbers are literals, derived in the
comments), and each "mutation" test shows that a plausible misreading -- no half-voxel
offset, the margin on the wrong side, border seeds on every face, an x/y swap -- fails it.
"""
import math

import numpy as np
import pytest

from oracle import hier_oracle as ho
from oracle import rw_oracle as ro

# ----------------------------------------------------------------------------- worked example
# Level l has Dl = 16 voxels per axis, bricks of s = 4, e = 1.5 -> s_e = floor(6.0) = 6, low
# margin ceil((6 - 4)/2) = 1, origins clamped to [0, Dl - s_e] = [0, 10] (R23):
#   brick 0 -> 0, 1 -> 3, 2 -> 7, 3 -> 11 -> 10.
# The parent level (8^3) holds the linear field P[z, y, x] = (x + 2y + 4z) / 49, so trilinear
# sampling is exact wherever the parent coordinate lies in [0, 7]:
#   child index i -> parent coordinate u(i) = (i + 0.5)/2 - 0.5 = i/2 - 0.25 (R25),
#   clamped: u(0) = 0 (from -0.25), u(15) = 7 (from 7.25).
DL, S, E = 16, 4, 1.5
SE = int(math.floor(E * S))
PAR = np.fromfunction(lambda z, y, x: (x + 2 * y + 4 * z) / 49.0, (8, 8, 8))


def _level_seeds(user=()):
    fx = np.zeros((DL, DL, DL), bool)
    val = np.zeros((DL, DL, DL))
    for (z, y, x), v in user:
        fx[z, y, x] = True
        val[z, y, x] = v
    return fx, val


def _check_worked_example():
    """Returns None if the oracle reproduces the hand-computed windows, else a message."""
    msgs = []
    # brick (bz, by, bx) = (0, 1, 2): origin (0, 3, 7), window = level [0,6) x [3,9) x [7,13).
    # Interior faces: all but z-low (the volume boundary, Neumann, reading c4).
    # A user fg seed at level (5, 5, 9) = window (5, 2, 2) sits on the z-high face: it wins.
    fx, val = _level_seeds([((5, 5, 9), 1.0)])
    w0, fixed, values, samp = ho.window_system(PAR, fx, val, (0, 1, 2), S, SE, DL)
    if list(w0) != [0, 3, 7]:
        return f"origin {w0} != [0, 3, 7]"
    # shell on 5 faces of a 6^3 cube: 6^3 - 5*4*4 = 136 voxels (the user seed is one of them)
    if int(fixed.sum()) != 136:
        msgs.append(f"{int(fixed.sum())} fixed voxels != 136")
    expect = {
        # window (z, y, x): (fixed, value) with value = (u_x + 2 u_y + 4 u_z) / 49
        (5, 0, 0): (True, (3.25 + 2 * 1.25 + 4 * 2.25) / 49),   # level (5,3,7)
        (0, 0, 3): (True, (4.75 + 2 * 1.25 + 4 * 0.0) / 49),    # level (0,3,10): y-low face
        (3, 5, 2): (True, (4.25 + 2 * 3.75 + 4 * 1.25) / 49),   # level (3,8,9): y-high face
        (1, 2, 5): (True, (5.75 + 2 * 2.25 + 4 * 0.25) / 49),   # level (1,5,12): x-high face
        (2, 3, 0): (True, (3.25 + 2 * 2.75 + 4 * 0.75) / 49),   # level (2,6,7): x-low face
        (5, 2, 2): (True, 1.0),                                  # user seed wins
        (0, 3, 3): (False, None),                                # z-low: volume boundary
        (2, 3, 3): (False, None),                                # interior
        (4, 1, 4): (False, None),                                # interior
    }
    for (z, y, x), (f, v) in expect.items():
        if bool(fixed[z, y, x]) != f:
            msgs.append(f"fixed{(z, y, x)} = {bool(fixed[z, y, x])}, expected {f}")
        elif f and abs(values[z, y, x] - v) > 1e-12:
            msgs.append(f"value{(z, y, x)} = {values[z, y, x]:.6f}, expected {v:.6f}")
    # initial guess: the parent sampled at every window voxel; (2, 3, 3) = level
    # (2, 6, 10): (4.75 + 2 * 2.75 + 4 * 0.75) / 49
    if abs(samp[2, 3, 3] - (4.75 + 5.5 + 3.0) / 49) > 1e-12:
        msgs.append(f"x0(2,3,3) = {samp[2, 3, 3]:.6f}")
    # brick (3, 3, 3): origin 10 on every axis (11 clamped), border seeds on the three low
    # faces only (10 + 6 = Dl: the high faces are the volume boundary)
    w0, fixed, values, _ = ho.window_system(PAR, *_level_seeds(), (3, 3, 3), S, SE, DL)
    if list(w0) != [10, 10, 10]:
        msgs.append(f"origin(3,3,3) {w0} != [10, 10, 10]")
    if not (fixed[0].all() and fixed[:, 0].all() and fixed[:, :, 0].all()
            and not fixed[1:, 1:, 1:].any()):
        msgs.append("brick (3,3,3): border seeds not exactly on the three low faces")
    # brick (0, 0, 0): origin 0, border seeds on the three high faces only; corner (5, 5, 5):
    # (2.25 + 2 * 2.25 + 4 * 2.25) / 49
    w0, fixed, values, _ = ho.window_system(PAR, *_level_seeds(), (0, 0, 0), S, SE, DL)
    if not (fixed[-1].all() and fixed[:, -1].all() and fixed[:, :, -1].all()
            and not fixed[:-1, :-1, :-1].any()):
        msgs.append("brick (0,0,0): border seeds not exactly on the three high faces")
    elif abs(values[5, 5, 5] - 15.75 / 49) > 1e-12:
        msgs.append(f"value(5,5,5) = {values[5, 5, 5]:.6f}")
    return "; ".join(msgs) or None


def test_border_seeds_worked_example():
    """sample_border on a hand-computed window: placement, faces, values."""
    assert _check_worked_example() is None, _check_worked_example()


def test_window_origins_worked_example():
    """Reading R23 with a margin that is not an integer: s = 4, e = 1.75 -> s_e = 7,
    margin ceil(1.5) = 2 on the low side, clamped to [0, Dl - s_e] = [0, 9] at Dl = 16."""
    assert [ho.window_origin(b, 4, 7, 16) for b in range(4)] == [0, 2, 6, 9]


@pytest.mark.parametrize("mutation", ["no_half_voxel", "margin_floor_plus_one",
                                      "no_margin", "all_faces", "swap_xy"])
def test_worked_example_catches_misreadings(monkeypatch, mutation):
    """Each plausible misreading of P:97-117 / R23-R25 changes the hand-computed window."""
    if mutation == "no_half_voxel":
        monkeypatch.setattr(ho, "parent_coord", lambda i: np.asarray(i, np.float64) / 2.0)
    elif mutation == "margin_floor_plus_one":
        monkeypatch.setattr(ho, "window_origin", lambda b, s, se, D: int(
            min(max(b * s - (se - s) // 2 - 1, 0), D - se)))
    elif mutation == "no_margin":
        monkeypatch.setattr(ho, "window_origin", lambda b, s, se, D: int(
            min(max(b * s, 0), D - se)))
    elif mutation == "all_faces":
        orig = ho.window_system

        def all_faces(P, fx, val, brick, s, se, Dl):
            w0, fixed, values, samp = orig(P, fx, val, brick, s, se, Dl)
            shell = np.ones((se, se, se), bool)
            shell[1:-1, 1:-1, 1:-1] = False
            border = shell & ~fx[tuple(slice(a, a + se) for a in w0)]
            return w0, fixed | border, np.where(border, samp, values), samp
        monkeypatch.setattr(ho, "window_system", all_faces)
    elif mutation == "swap_xy":
        orig_s = ho.sample_parent
        monkeypatch.setattr(ho, "sample_parent", lambda P, zs, ys, xs: orig_s(
            np.swapaxes(P, 1, 2), zs, ys, xs))
    assert _check_worked_example() is not None


# ----------------------------------------------------------------------------- whole volume
def _blob_volume(D, seed, nseed):
    """Three bright blobs (0.8) on 0.2 + N(0, 0.03), u16; nseed fg seeds inside the blobs and
    nseed bg seeds outside (scribble-like point sets)."""
    rng = np.random.default_rng([31, seed])
    z, y, x = np.meshgrid(*(np.arange(D),) * 3, indexing="ij")
    inside = np.zeros((D, D, D), bool)
    for _ in range(3):
        c = rng.uniform(0.25, 0.75, 3) * D
        r = rng.uniform(0.12, 0.2) * D
        inside |= (z - c[0]) ** 2 + (y - c[1]) ** 2 + (x - c[2]) ** 2 < r * r
    g = np.clip(np.where(inside, 0.8, 0.2) + rng.normal(0, 0.03, (D, D, D)), 0, 1)
    seeds = np.zeros((D, D, D), np.uint8)
    seeds.ravel()[rng.choice(np.flatnonzero(inside.ravel()), nseed, replace=False)] = 1
    seeds.ravel()[rng.choice(np.flatnonzero(~inside.ravel()), nseed, replace=False)] = 2
    return np.rint(g * 65535).astype(np.uint16), seeds


@pytest.mark.parametrize("seed", [0, 1])
def test_hierarchical_approximates_full_volume_solve(seed):
    """each level's solution approximates the random walker "computed on the full
    volume"; Octree Dice ~ Basic.  D = 64, s = 16, e = 1.25 (three levels, windows with
    interior faces on every level below the root), no pruning.  Bound (DESIGN.md §3 R30):
    labels agree on >= 99.5 % of voxels; mean |dp| <= 0.05 (measured 0.02-0.03: the coarse
    levels see 8x / 64x larger seed voxels, so probabilities away from edges shift while the
    p = 0.5 surface stays on the intensity edge)."""
    vol, seeds = _blob_volume(64, seed, 200)
    o = ho.hier_segment(vol, seeds, s=16, e=1.25, beta=100.0, tol=1e-10, prune=False)
    g = ro.normalise(vol, 1 / 65535, 0.0)
    fixed, val = ho.seeds_from_bits(ho.seed_bits(seeds))
    ref = ro.solve_brick(g, fixed, val, 100.0, 1e-6, tol=1e-10)
    p = np.where(fixed, val, np.clip(ref["x"], 0, 1))
    assert len(o["stats"]) == 3 and all(st["solved"] > 0 for st in o["stats"])
    agree = np.mean((o["prob"] > 0.5) == (p > 0.5))
    assert agree >= 0.995, agree
    assert np.mean(np.abs(o["prob"] - p)) <= 0.05


@pytest.mark.parametrize("profile", ["uniform", "smooth"])
def test_hierarchical_tracks_series_resistor_ramp(profile):
    """Layered volume (g depends on x only), fg seeds on the plane x = 0, bg on x = D - 1:
    the full-volume solution is the 1-D series-resistor ramp p(x) = sum_{k>=x} 1/w_k /
    sum_k 1/w_k (SURVEY §8(c) closed forms).  The hierarchical field must track the ramp
    within 1 / (2 (D_root - 1)) = 0.033 everywhere: the root ramp differs from the fine one
    by at most half a root-voxel slope, and every window solve only interpolates between its
    border values (discrete maximum principle), so the error cannot grow level to level
    (DESIGN.md §3 R30).  (It is not exactly constant over y / z: windows whose y / z faces are
    interior carry parent samples there, windows on the volume border are Neumann.)"""
    D, s = 64, 16
    xs = np.arange(D)
    gx = np.full(D, 0.5) if profile == "uniform" else 0.5 + 0.3 * np.sin(2 * np.pi * xs / D)
    vol = np.rint(np.broadcast_to(gx, (D, D, D)) * 65535).astype(np.uint16)
    seeds = np.zeros((D, D, D), np.uint8)
    seeds[:, :, 0] = 1
    seeds[:, :, D - 1] = 2
    beta = 10.0
    gq = vol[0, 0, :] / 65535.0
    inv = 1.0 / (np.exp(-beta * np.diff(gq) ** 2) + 1e-6)
    ramp = np.array([inv[i:].sum() for i in range(D)]) / inv.sum()
    o = ho.hier_segment(vol, seeds, s=s, e=1.25, beta=beta, tol=1e-11, prune=False)
    p = o["prob"]
    err = np.abs(p - ramp[None, None, :]).max()
    assert err <= 1.0 / (2 * (s - 1)), err
