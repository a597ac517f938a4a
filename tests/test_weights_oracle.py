"""Pins of oracle/weights_oracle.py (the paper's alternative weights,
P:123-133) against things other than the oracle itself: the paper's/SPEC's worked values,
brute-force loops, an independent library (scipy.stats) and invariances."""
import itertools
import math

import numpy as np
import pytest
import scipy.stats

from oracle import weights_oracle as wo
from oracle import rw_oracle as ro
from conftest import read_golden

EPS = 1e-6


def test_poisson_golden_values():
    """S:190 / P:133 worked values."""
    for n_p, n_q, want in read_golden("poisson_weight.txt"):
        counts = np.array([[[float(n_p), float(n_q)]]])
        W = wo.poisson_planes(counts, 0.0)
        assert W[0, 0, 0, 0] == pytest.approx(float(want), rel=1e-12)
        assert W[0, 0, 0, 1] == 0.0          # no edge leaves the brick (reading c4)


def test_poisson_counts_and_symmetry():
    rng = np.random.default_rng(0)
    v = rng.integers(0, 5000, (3, 4, 5)).astype(np.uint16)
    c = wo.poisson_counts(v, 2.0)
    assert np.array_equal(c, v.astype(np.float64) * 2.0)
    assert (wo.poisson_counts(np.array([-5, 3], np.int16)) == [0.0, 3.0]).all()
    W = wo.poisson_planes(c, EPS)
    Wr = wo.poisson_planes(c[:, :, ::-1], EPS)       # mirror x: same edge set, reversed
    np.testing.assert_array_equal(W[0][:, :, :-1], Wr[0][:, :, :-1][:, :, ::-1])


def test_gaussian_sigma2_brute_force():
    """sigma^2 = mean squared 6-neighbour difference, by an explicit double loop."""
    rng = np.random.default_rng(1)
    g = rng.uniform(0, 1, (3, 4, 5))
    nz, ny, nx = g.shape
    tot, cnt = 0.0, 0
    for z, y, x in itertools.product(range(nz), range(ny), range(nx)):
        for dz, dy, dx in ((0, 0, 1), (0, 1, 0), (1, 0, 0)):
            if z + dz < nz and y + dy < ny and x + dx < nx:
                tot += (g[z + dz, y + dy, x + dx] - g[z, y, x]) ** 2
                cnt += 1
    assert wo.gaussian_sigma2(g) == pytest.approx(tot / cnt, rel=1e-13)
    W = wo.gaussian_planes(g, 0.0)
    z, y, x = 1, 2, 3
    assert W[1, z, y, x] == pytest.approx(math.exp(-(g[z, y + 1, x] - g[z, y, x]) ** 2 / (2 * tot / cnt)))


def test_gaussian_scale_invariance_and_constant():
    """The weight depends on differences relative to their own spread: g -> c g + d leaves
    it unchanged; a constant brick has sigma^2 = floor and every weight 1 (+eps)."""
    rng = np.random.default_rng(2)
    g = rng.uniform(0, 1, (4, 5, 6))
    np.testing.assert_allclose(wo.gaussian_planes(3.0 * g + 0.25, EPS), wo.gaussian_planes(g, EPS),
                               rtol=1e-12)
    W = wo.gaussian_planes(np.full((3, 3, 4), 0.4), EPS)
    assert wo.gaussian_sigma2(np.full((3, 3, 4), 0.4)) == wo.SIGMA2_FLOOR
    assert np.allclose(W[0][:, :, :-1], 1.0 + EPS) and np.all(W[0][:, :, -1] == 0)


def test_ttest_stats_match_brute_force_neighbourhoods():
    """Neighbourhood sizes, means and unbiased variances by explicit per-voxel loops."""
    rng = np.random.default_rng(3)
    g = rng.uniform(0, 1, (4, 5, 6))
    N, M, V = wo.ttest_stats(g, 1)
    nz, ny, nx = g.shape
    for z, y, x in [(0, 0, 0), (1, 2, 3), (3, 4, 5), (0, 2, 5)]:
        vals = [g[zz, yy, xx] for zz in range(z - 1, z + 2) for yy in range(y - 1, y + 2)
                for xx in range(x - 1, x + 2) if 0 <= zz < nz and 0 <= yy < ny and 0 <= xx < nx]
        assert N[z, y, x] == len(vals)
        assert M[z, y, x] == pytest.approx(np.mean(vals), rel=1e-13)
        assert V[z, y, x] == pytest.approx(np.var(vals, ddof=1), rel=1e-12)
    assert N[0, 0, 0] == 8 and N[1, 2, 3] == 27     # corner clipped to 2^3


def test_ttest_against_scipy_welch():
    """Welch's t of the two neighbourhoods equals scipy.stats.ttest_ind(equal_var=False), and
    the weight is its two-tailed normal p-value 2 (1 - Phi(|t|)) (+eps)."""
    rng = np.random.default_rng(4)
    g = rng.uniform(0, 1, (5, 5, 5)) + np.arange(5)[None, None, :] * 0.05
    W = wo.ttest_planes(g, EPS, 1)
    for (z, y, x), ax in [((2, 2, 2), 0), ((1, 3, 0), 1), ((0, 0, 0), 2)]:
        q = (z + (ax == 2), y + (ax == 1), x + (ax == 0))
        def hood(c):
            cz, cy, cx = c
            return [g[a, b, d] for a in range(cz - 1, cz + 2) for b in range(cy - 1, cy + 2)
                    for d in range(cx - 1, cx + 2) if 0 <= a < 5 and 0 <= b < 5 and 0 <= d < 5]
        t = scipy.stats.ttest_ind(hood((z, y, x)), hood(q), equal_var=False).statistic
        N, M, V = wo.ttest_stats(g, 1)
        tw = wo.welch_t(M[z, y, x], V[z, y, x], N[z, y, x], M[q], V[q], N[q])
        assert tw == pytest.approx(t, rel=1e-10)
        assert W[ax, z, y, x] == pytest.approx(2 * scipy.stats.norm.sf(abs(t)) + EPS, rel=1e-10)


def test_ttest_flat_and_shift_invariance():
    """two flat identical neighbourhoods -> P-value 1 (weight 1 + eps); adding a
    constant to every voxel changes nothing; a step edge gets a tiny weight."""
    W = wo.ttest_planes(np.full((3, 4, 5), 0.3), EPS, 1)
    assert np.allclose(W[0][:, :, :-1], 1.0 + EPS)
    rng = np.random.default_rng(5)
    g = rng.uniform(0, 1, (4, 4, 4))
    np.testing.assert_allclose(wo.ttest_planes(g + 0.125, EPS), wo.ttest_planes(g, EPS), rtol=1e-10)
    step = np.zeros((4, 4, 8))
    step[:, :, 4:] = 1.0
    step += rng.normal(0, 0.01, step.shape)
    Ws = wo.ttest_planes(step, EPS, 1)
    row = Ws[0, 2, 2, :-1]
    # every edge whose 3^3 neighbourhoods straddle the step (x = 2..4) is weak, the others not
    assert row[2:5].max() < 0.05 < row[[0, 1, 5, 6]].min()


def test_planes_to_edges_roundtrip_and_solve():
    """planes_to_edges gives rw_oracle's own edge list for Grady planes (same order), so a
    solve with externally supplied weights is the ordinary solve."""
    rng = np.random.default_rng(6)
    g = rng.uniform(0, 1, (3, 4, 5))
    i, j, w = ro.edge_list(g, 30.0, EPS)
    i2, j2, w2 = wo.planes_to_edges(ro.weight_planes(g, 30.0, EPS))
    assert np.array_equal(i, i2) and np.array_equal(j, j2)
    np.testing.assert_allclose(w, w2, rtol=1e-15)
    fixed = np.zeros(g.size, bool)
    fixed[[0, g.size - 1]] = True
    xs = np.zeros(g.size)
    xs[0] = 1.0
    a = ro.solve_brick(g, fixed, xs, 30.0, EPS)
    b = ro.solve_brick(g, fixed, xs, 30.0, EPS, edges=(i2, j2, w2))
    np.testing.assert_allclose(a["x"], b["x"], atol=1e-12)
