"""Pins of oracle/hier_oracle.py (the hierarchical driver of P:83-161)
against closed forms, brute force and the plain random walker it must reduce to."""
import itertools

import numpy as np
import pytest

from oracle import hier_oracle as ho
from oracle import rw_oracle as ro
import workloads as wl


def small_volume(D, seed, nblob=2):
    """Seeded u16 volume with blobs + noise and a label volume (1 fg inside the first blob,
    2 bg near the corners)."""
    rng = np.random.default_rng([21, seed])
    z, y, x = np.meshgrid(*(np.arange(D),) * 3, indexing="ij")
    g = np.full((D, D, D), 0.2)
    cs = []
    for _ in range(nblob):
        c = rng.uniform(0.3, 0.7, 3) * D
        r = rng.uniform(0.15, 0.25) * D
        g[(z - c[0]) ** 2 + (y - c[1]) ** 2 + (x - c[2]) ** 2 < r * r] = 0.8
        cs.append(c)
    g = np.clip(g + rng.normal(0, 0.03, g.shape), 0, 1)
    vol = np.rint(g * 65535).astype(np.uint16)
    seeds = np.zeros((D, D, D), np.uint8)
    c = np.round(cs[0]).astype(int)
    seeds[c[0], c[1], c[2]] = 1
    seeds[c[0], c[1], min(c[2] + 1, D - 1)] = 1
    seeds[1, 1, 1] = seeds[D - 2, D - 2, D - 2] = seeds[1, D - 2, 1] = 2
    return vol, seeds


def multi_volume(D, seed, K=3):
    """Seeded u16 volume with K-1 blobs + noise and multi-class labels: class k seeds at the
    centre of blob k, class K (background) near the corners."""
    rng = np.random.default_rng([23, seed])
    z, y, x = np.meshgrid(*(np.arange(D),) * 3, indexing="ij")
    g = np.full((D, D, D), 0.15)
    labels = np.zeros((D, D, D), np.uint8)
    for k in range(1, K):
        c = rng.uniform(0.3, 0.7, 3) * D
        r = rng.uniform(0.12, 0.2) * D
        g[(z - c[0]) ** 2 + (y - c[1]) ** 2 + (x - c[2]) ** 2 < r * r] = 0.3 + 0.5 * k / K
        cs = np.round(c).astype(int)
        labels[cs[0], cs[1], cs[2]] = k
        labels[cs[0], cs[1], min(cs[2] + 1, D - 1)] = k
    g = np.clip(g + rng.normal(0, 0.03, g.shape), 0, 1)
    labels[1, 1, 1] = labels[D - 2, D - 2, D - 2] = labels[1, D - 2, 1] = K
    return np.rint(g * 65535).astype(np.uint16), labels


def test_multiclass_fields_partition_seeds():
    """K = 3 on a 3-level volume.  Without pruning every class field keeps its own seeds at 1
    and the other classes' seeds at 0 (P:107 one-vs-rest), so each seed voxel gets its own
    class from the argmax; with H_p, dt pruning never fires and a pruned brick
    carries its ancestor's field (R26), so seeds there are only approximately kept."""
    vol, lab = multi_volume(32, 3)
    o = ho.hier_segment_labels(vol, lab, 3, s=8, e=1.5, beta=50.0, tol=1e-9, prune=False)
    for k in range(3):
        assert np.all(o["prob"][k][lab == k + 1] == 1.0)
        assert np.all(o["prob"][k][(lab > 0) & (lab != k + 1)] == 0.0)
    assert np.array_equal(o["labels"][lab > 0], lab[lab > 0])
    p = ho.hier_segment_labels(vol, lab, 3, s=8, e=1.5, beta=50.0, tol=1e-9, t_hom=0.3)
    assert all(st["pruned_dt"] == 0 for k in range(3) for st in p["stats"][k])
    assert sum(st["pruned_hom"] for k in range(3) for st in p["stats"][k]) > 0


def test_single_level_is_the_plain_random_walker():
    """Eq. 1: D = s -> the root solve of the whole volume."""
    vol, seeds = small_volume(16, 0)
    o = ho.hier_segment(vol, seeds, s=16, e=1.25, beta=50.0)
    g = ro.normalise(vol, 1 / 65535, 0.0)
    fixed, val = ho.seeds_from_bits(ho.seed_bits(seeds))
    ref = ro.solve_brick(g, fixed, val, 50.0, 1e-6)
    np.testing.assert_allclose(o["prob"], np.where(fixed, val, np.clip(ref["x"], 0, 1)), atol=1e-12)


def test_whole_level_window_reduces_to_plain_solve():
    """e = 2, D = 2s: the level-0 window is the whole level (no interior faces, so no border
    seeds) -> the unique plain random walker solution, whatever the initial guess."""
    vol, seeds = small_volume(16, 1)
    o = ho.hier_segment(vol, seeds, s=8, e=2.0, beta=50.0, prune=False)
    g = ro.normalise(vol, 1 / 65535, 0.0)
    fixed, val = ho.seeds_from_bits(ho.seed_bits(seeds))
    ref = ro.solve_brick(g, fixed, val, 50.0, 1e-6)
    np.testing.assert_allclose(o["prob"], np.where(fixed, val, np.clip(ref["x"], 0, 1)), atol=1e-8)


def test_trilinear_sampling_closed_forms():
    """constant -> constant; linear ramp -> the same ramp at interior child
    voxel centres; 2^3 one-hot parent -> hand-evaluated weights."""
    P = np.full((4, 4, 4), 0.9)
    assert np.allclose(ho.upsample(P, (8, 8, 8)), 0.9)
    px = np.arange(4, dtype=float)
    R = np.broadcast_to(0.1 * px, (4, 4, 4))
    U = ho.upsample(R, (8, 8, 8))
    for i in range(1, 7):                      # interior: child centre (i+0.5)/2 - 0.5
        assert U[3, 3, i] == pytest.approx(0.1 * ((i + 0.5) / 2 - 0.5))
    C = np.zeros((2, 2, 2))
    C[0, 0, 0] = 1.0
    U = ho.upsample(C, (4, 4, 4))
    f = {0: 1.0, 1: 0.75, 2: 0.25, 3: 0.0}     # weight of parent 0 at child i (clamped)
    for z, y, x in itertools.product(range(4), repeat=3):
        assert U[z, y, x] == pytest.approx(f[z] * f[y] * f[x])


def test_seed_pyramid_conflicts_brute_force():
    rng = np.random.default_rng(3)
    seeds = rng.choice([0, 0, 0, 1, 2], size=(8, 8, 8)).astype(np.uint8)
    pyr = ho.seed_bit_pyramid(seeds, 3)
    for l, b in enumerate(pyr):
        n = 8 >> l
        for z, y, x in itertools.product(range(n), repeat=3):
            blk = seeds[z << l:(z + 1) << l, y << l:(y + 1) << l, x << l:(x + 1) << l]
            want = (1 if (blk == 1).any() else 0) | (2 if (blk == 2).any() else 0)
            assert b[z, y, x] == want
    fixed, val = ho.seeds_from_bits(np.array([0, 1, 2, 3], np.uint8))
    assert fixed.tolist() == [False, True, True, False] and val.tolist() == [0, 1, 0, 0]


def test_window_origin():
    """Reading R23: margin ceil((se-s)/2) low side, shifted inside, always covering the brick."""
    s, se = 32, 40
    assert ho.window_origin(3, s, se, 256) == 3 * 32 - 4
    assert ho.window_origin(0, s, se, 256) == 0
    assert ho.window_origin(7, s, se, 256) == 256 - 40
    for D in (64, 128):
        for b in range(D // s):
            o = ho.window_origin(b, s, se, D)
            assert 0 <= o <= b * s and b * s + s <= o + se <= D


def test_constant_parent_gives_constant_children():
    """All seeds foreground -> the root field is 1 and every border seed and solution is 1."""
    vol, seeds = small_volume(32, 2)
    seeds[seeds > 0] = 1
    o = ho.hier_segment(vol, seeds, s=8, e=1.25, beta=50.0, prune=False)
    assert np.allclose(o["prob"], 1.0, atol=1e-8)


def test_pruning_soundness_against_unpruned():
    """P:139-161 / S:321: pruned_dt regions threshold like the unpruned run, pruned_hom
    regions stay within t_hom (+ interpolation slack) of it; pruning solves fewer bricks."""
    vol, seeds = small_volume(32, 4)
    full = ho.hier_segment(vol, seeds, s=8, e=1.25, beta=50.0, tol=1e-8, prune=False)
    pr = ho.hier_segment(vol, seeds, s=8, e=1.25, beta=50.0, tol=1e-8, prune=True)
    assert sum(st["solved"] for st in pr["stats"]) < sum(st["solved"] for st in full["stats"])
    assert np.abs(pr["prob"] - full["prob"]).max() < 0.3 + 0.05
    agree = ((pr["prob"] > 0.5) == (full["prob"] > 0.5)).mean()
    assert agree > 0.99


def test_incremental_noop_identity():
    """S:360 / P:175-181: re-running with unchanged labels reuses the root's subtree: the
    output equals the previous output voxel for voxel."""
    vol, seeds = small_volume(32, 5)
    first = ho.hier_segment(vol, seeds, s=8, e=1.5, beta=50.0, tol=1e-9)
    again = ho.hier_segment(vol, seeds, s=8, e=1.5, beta=50.0, tol=1e-9, prev=first)
    assert again["stats"][-1]["reused"] == 1
    assert sum(st["solved"] for st in again["stats"]) == 1      # only the root is re-solved
    assert np.array_equal(again["prob"], first["prob"])


def test_incremental_new_seed_matches_full_recompute():
    """one new foreground seed where the solution is already highest (inside the
    labelled foreground): coarse levels barely change, so subtrees are reused and far fewer
    bricks are solved; the result agrees with a full run on the new labels."""
    vol, seeds = small_volume(32, 6)
    first = ho.hier_segment(vol, seeds, s=8, e=1.5, beta=50.0, tol=1e-9)
    new = seeds.copy()
    p = np.where(seeds > 0, -1.0, first["prob"])
    new[np.unravel_index(np.argmax(p), p.shape)] = 1
    inc = ho.hier_segment(vol, new, s=8, e=1.5, beta=50.0, tol=1e-9, prev=first)
    full = ho.hier_segment(vol, new, s=8, e=1.5, beta=50.0, tol=1e-9)
    assert sum(st["solved"] for st in inc["stats"]) < sum(st["solved"] for st in full["stats"])
    assert np.abs(inc["prob"] - full["prob"]).max() < 0.3
    assert ((inc["prob"] > 0.5) == (full["prob"] > 0.5)).mean() > 0.99


def test_incremental_conflict_vetoes_reuse():
    """A changed label that creates a seed conflict in the root brick ("conflicts where
    at least one of the recently added labels is involved") forces a recomputation."""
    vol, seeds = small_volume(32, 7)
    first = ho.hier_segment(vol, seeds, s=8, e=1.5, beta=50.0, tol=1e-9)
    new = seeds.copy()
    new[0, 0, 0], new[0, 0, 1] = 1, 2           # fg + bg in one root voxel: a new conflict
    inc = ho.hier_segment(vol, new, s=8, e=1.5, beta=50.0, tol=1e-9, prev=first)
    assert inc["stats"][-1]["reused"] == 0 and inc["stats"][-1]["conflict"] == 1


def test_multiclass_two_classes_is_the_binary_run():
    """K = 2: class 1's probability is the binary run with class-1 seeds foreground; the
    argmax labels agree with thresholding the binary field at 0.5 wherever the two class
    fields are not tied."""
    vol, seeds = small_volume(32, 8)
    lab = np.where(seeds == 1, 1, np.where(seeds == 2, 2, 0)).astype(np.uint8)
    mc = ho.hier_segment_labels(vol, lab, 2, s=8, e=1.5, beta=50.0, tol=1e-9)
    bi = ho.hier_segment(vol, seeds, s=8, e=1.5, beta=50.0, tol=1e-9, t_bin=-1.0)
    np.testing.assert_allclose(mc["prob"][0], bi["prob"], atol=1e-12)
    sure = np.abs(mc["prob"][0] - mc["prob"][1]) > 1e-6
    assert np.array_equal((mc["labels"] == 1)[sure], (mc["prob"][0] > mc["prob"][1])[sure])
    assert set(np.unique(mc["labels"])) <= {1, 2}
