"""Pins of the hierarchical oracle on volumes that are not cubic and not s 2^k (P:109-111:
"the proposed method is not restricted to volumes of size 2^i s ... bricks at the border of
the volume may be smaller than s^3 voxels"; reading R31 in DESIGN.md §3).  The in-HBM GPU
driver takes cubic s 2^k volumes; rw_hier_segment_ooc takes any dims and is checked against
this oracle (tests/test_gpu_hier_ooc.py)."""
import numpy as np
import pytest

from oracle import hier_oracle as ho
from oracle import rw_oracle as ro


def test_level_dims_and_root():
    """Level dims are the pyramid's ceil(d/2) (c12); the root is the first level whose
    dims are all <= s; cubic s 2^k volumes keep their k + 1 levels."""
    assert ho.level_dims((40, 56, 72), 16) == [(40, 56, 72), (20, 28, 36), (10, 14, 18), (5, 7, 9)]
    assert ho.level_dims((64, 64, 64), 16) == [(64, 64, 64), (32, 32, 32), (16, 16, 16)]
    assert ho.level_dims((16, 64, 33), 16) == [(16, 64, 33), (8, 32, 17), (4, 16, 9)]
    assert ho.level_dims((12, 8, 16), 16) == [(12, 8, 16)]          # one brick: the root


def test_window_origin_narrow_level():
    """R23 + R31: a window never leaves the level; a level narrower than s_e is taken whole."""
    assert ho.window_origin(0, 16, 20, 14) == 0        # side min(20, 14) = 14 -> [0, 14)
    assert ho.window_origin(1, 16, 20, 18) == 0        # side 18 -> whole axis
    assert ho.window_origin(2, 16, 20, 36) == 16       # shifted inward: 36 - 20
    assert ho.window_origin(1, 16, 20, 36) == 14       # 16 - ceil(4/2)
    w0, fixed, values, samp = ho.window_system(
        np.full((3, 4, 5), 0.5), np.zeros((5, 7, 9), bool), np.zeros((5, 7, 9)), (0, 0, 0),
        4, 6, (5, 7, 9))
    assert fixed.shape == (5, 6, 6) and w0 == [0, 0, 0]
    # z is taken whole (both z faces on the volume boundary: Neumann); the high y / x faces
    # are interior and carry parent samples
    assert not fixed[1:-1, :-1, :-1].any()
    assert fixed[:, -1, :].all() and fixed[:, :, -1].all()


def _ragged_volume(shape, seed, nseed):
    rng = np.random.default_rng([37, seed])
    z, y, x = np.meshgrid(*(np.arange(n) for n in shape), indexing="ij")
    inside = np.zeros(shape, bool)
    for _ in range(3):
        c = rng.uniform(0.25, 0.75, 3) * np.array(shape)
        r = rng.uniform(0.12, 0.2) * min(shape)
        inside |= (z - c[0]) ** 2 + (y - c[1]) ** 2 + (x - c[2]) ** 2 < r * r
    g = np.clip(np.where(inside, 0.8, 0.2) + rng.normal(0, 0.03, shape), 0, 1)
    seeds = np.zeros(shape, np.uint8)
    seeds.ravel()[rng.choice(np.flatnonzero(inside.ravel()), nseed, replace=False)] = 1
    seeds.ravel()[rng.choice(np.flatnonzero(~inside.ravel()), nseed, replace=False)] = 2
    return np.rint(g * 65535).astype(np.uint16), seeds


@pytest.mark.parametrize("shape", [(40, 56, 72), (36, 64, 48)])
def test_ragged_hierarchical_approximates_full_volume_solve(shape):
    """As the cubic pin (R30 b) on ragged non-cubic volumes, s = 16, e = 1.25: every level
    below the root has smaller border bricks; labels agree with the whole-volume random
    walker on >= 99.5 % of voxels, mean |dp| <= 0.05."""
    vol, seeds = _ragged_volume(shape, 0, 150)
    o = ho.hier_segment(vol, seeds, s=16, e=1.25, beta=100.0, tol=1e-10, prune=False)
    assert o["prob"].shape == shape
    g = ro.normalise(vol, 1 / 65535, 0.0)
    fixed, val = ho.seeds_from_bits(ho.seed_bits(seeds))
    ref = ro.solve_brick(g, fixed, val, 100.0, 1e-6, tol=1e-10)
    p = np.where(fixed, val, np.clip(ref["x"], 0, 1))
    assert all(st["solved"] > 0 for st in o["stats"])
    agree = np.mean((o["prob"] > 0.5) == (p > 0.5))
    assert agree >= 0.995, agree
    assert np.mean(np.abs(o["prob"] - p)) <= 0.05


def test_ragged_tracks_series_resistor_ramp():
    """Layered ragged volume (g depends on x only; fg plane x = 0, bg plane x = nx - 1): the
    whole-volume solution is the series-resistor ramp; the hierarchical field tracks it within
    half a root-voxel slope, 1 / (2 (nx_root - 1)) (R30 c), with border bricks of 8 / 4 / 2
    voxels along x at the three levels below the root."""
    shape, s = (24, 40, 72), 16
    nx = shape[2]
    xs = np.arange(nx)
    gx = 0.5 + 0.3 * np.sin(2 * np.pi * xs / nx)
    vol = np.rint(np.broadcast_to(gx, shape) * 65535).astype(np.uint16)
    seeds = np.zeros(shape, np.uint8)
    seeds[:, :, 0] = 1
    seeds[:, :, nx - 1] = 2
    beta = 10.0
    gq = vol[0, 0, :] / 65535.0
    inv = 1.0 / (np.exp(-beta * np.diff(gq) ** 2) + 1e-6)
    ramp = np.array([inv[i:].sum() for i in range(nx)]) / inv.sum()
    o = ho.hier_segment(vol, seeds, s=s, e=1.25, beta=beta, tol=1e-11, prune=False)
    nx_root = ho.level_dims(shape, s)[-1][2]
    err = np.abs(o["prob"] - ramp[None, None, :]).max()
    assert err <= 1.0 / (2 * (nx_root - 1)), (err, nx_root)


def test_ragged_seed_pyramid_bruteforce():
    """OR over the present children at odd dims, by brute force (R22 + R31)."""
    rng = np.random.default_rng(5)
    seeds = rng.choice(np.array([0, 0, 0, 1, 2], np.uint8), size=(5, 7, 9))
    b = ho.seed_bit_pyramid(seeds, 3)
    assert [x.shape for x in b] == [(5, 7, 9), (3, 4, 5), (2, 2, 3)]
    for l in (1, 2):
        lo, hi = b[l - 1], b[l]
        for Z, Y, X in np.ndindex(hi.shape):
            acc = 0
            for z in (2 * Z, 2 * Z + 1):
                for y in (2 * Y, 2 * Y + 1):
                    for x in (2 * X, 2 * X + 1):
                        if z < lo.shape[0] and y < lo.shape[1] and x < lo.shape[2]:
                            acc |= int(lo[z, y, x])
            assert hi[Z, Y, X] == acc
