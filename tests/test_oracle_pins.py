"""Pins of the fp64 oracle against facts fixed by the paper and by mathematics (CPU only).

Each test names the plausible oracle mistake it would catch.
"""
import math

import numpy as np
import pytest

from conftest import read_golden
from oracle import rw_oracle as ro
from oracle import energy
import workloads as wl
from workloads import gen


# ------------------------------------------------------------------ weights
def test_weight_closed_form_values():
    """Delta = 0 -> exp(0) + eps; beta*Delta^2 = 1 -> e^-1 + eps.  Catches a dropped
    eps, a missing square, a wrong sign in the exponent or beta applied twice."""
    g = np.array([[[0.2, 0.2, 0.3, 0.1]]])           # nz=ny=1, nx=4
    i, j, w = ro.edge_list(g, beta=100.0, eps=1e-6)
    assert list(i) == [0, 1, 2] and list(j) == [1, 2, 3]
    assert w[0] == pytest.approx(1.0 + 1e-6, abs=1e-15)
    assert w[1] == pytest.approx(math.e ** -1 + 1e-6, rel=1e-12)
    assert w[2] == pytest.approx(math.exp(-100 * 0.04) + 1e-6, rel=1e-12)


def test_weight_planes_layout_and_faces():
    """W_a[v] = w(v, v+e_a), zero on the + face (reading c4).  Catches axis transposition and
    off-by-one face handling: compared with an explicit per-voxel loop."""
    rng = np.random.default_rng(1)
    g = rng.uniform(0, 1, (3, 4, 5))
    W = ro.weight_planes(g, 7.0, 1e-6)
    nz, ny, nx = g.shape
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                for a, (dx, dy, dz) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
                    X, Y, Z = x + dx, y + dy, z + dz
                    exp = (math.exp(-7.0 * (g[Z, Y, X] - g[z, y, x]) ** 2) + 1e-6
                           if (X < nx and Y < ny and Z < nz) else 0.0)
                    assert W[a, z, y, x] == pytest.approx(exp, rel=1e-13, abs=0)


def test_edge_list_matches_bruteforce_enumeration():
    """Vectorised edge enumeration == the pure-Python neighbour loop (energy.py)."""
    rng = np.random.default_rng(2)
    g = rng.uniform(0, 1, (3, 4, 5))
    i, j, w = ro.edge_list(g, 30.0, 1e-6)
    e2 = energy.grid_edges(5, 4, 3)
    w2 = energy.weights(list(g.ravel()), e2, 30.0, 1e-6)
    a = sorted(zip(i.tolist(), j.tolist(), w.tolist()))
    b = sorted((p, q, ww) for (p, q), ww in zip(e2, w2))
    assert len(a) == len(b) == 3 * 4 * 4 + 3 * 3 * 5 + 2 * 4 * 5
    for (p, q, x), (p2, q2, y) in zip(a, b):
        assert (p, q) == (p2, q2) and x == pytest.approx(y, rel=1e-14)


def test_weight_symmetry_under_mirroring():
    """Mirroring the brick along x mirrors the x-weights."""
    rng = np.random.default_rng(3)
    g = rng.uniform(0, 1, (2, 3, 6))
    W = ro.weight_planes(g, 50.0, 1e-6)
    Wm = ro.weight_planes(g[:, :, ::-1], 50.0, 1e-6)
    np.testing.assert_allclose(Wm[0, :, :, :-1], W[0, :, :, :-1][:, :, ::-1], rtol=1e-14)


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("name", ["chain3.txt", "chain5.txt"])
def test_golden_chain(name):
    """SPEC S:211-212 worked examples: uniform chains -> exact linear interpolation."""
    g, f, v, x = read_golden(name)
    g = np.array(g, float)[None, None, :]
    o = ro.solve_brick(g, np.array(f, int), np.array(v, float), 100.0, 1e-6)
    np.testing.assert_allclose(o["x"].ravel(), np.array(x, float), atol=1e-12)


def test_chain_series_resistor():
    """Arbitrary-weight chain: x_i = sum_{k>=i} 1/w_k / sum_k 1/w_k (edge k joins k, k+1).
    Catches a wrong diagonal, a wrong sign of b, or a swapped i/j in assembly."""
    rng = np.random.default_rng(4)
    n = 17
    g = rng.uniform(0, 1, n)
    beta, eps = 20.0, 1e-6
    w = np.array([math.exp(-beta * (g[k + 1] - g[k]) ** 2) + eps for k in range(n - 1)])
    R = 1.0 / w
    expect = np.array([R[i:].sum() / R.sum() for i in range(n)])
    f = np.zeros(n, int); f[[0, -1]] = 1
    v = np.zeros(n); v[0] = 1.0
    o = ro.solve_brick(g[None, None, :], f, v, beta, eps)
    np.testing.assert_allclose(o["x"].ravel(), expect, atol=1e-11)


def test_layered_volume_reduces_to_chain():
    """g depends on x only, x=0 plane = 1, x=nx-1 plane = 0: every yz plane is constant and
    equals the 1D series-resistor value (exercises y/z Neumann faces, reading c4)."""
    p = wl.layered(9, 4, 3, seed=5)
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    o = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps)
    x = o["x"]
    gx = g[0, 0, :]
    w = np.exp(-p.beta * np.diff(gx) ** 2) + p.eps
    R = 1.0 / w
    expect = np.array([R[i:].sum() / R.sum() for i in range(len(gx))])
    np.testing.assert_allclose(x, np.broadcast_to(expect, x.shape), atol=1e-10)


def test_constant_solution():
    """All fixed values = c -> x = c everywhere (harmonic with constant boundary)."""
    p = wl.random_brick(6, 5, 4, seed=6, nseed=10)
    p.values[:] = 0.37
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    o = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps)
    np.testing.assert_allclose(o["x"], 0.37, atol=1e-11)


# ------------------------------------------------------------------ brute force / dense
@pytest.mark.parametrize("seed,dims,cont", [(10, (4, 3, 3), False), (11, (3, 4, 4), True),
                                            (12, (5, 3, 2), True), (13, (2, 2, 6), False)])
def test_oracle_equals_energy_minimiser(seed, dims, cont):
    """Oracle PCG solution == exact minimiser of the brute-force Dirichlet energy,
    built only from point evaluations of D.  Pins assembly + b + CG together."""
    nx, ny, nz = dims
    p = wl.random_brick(nx, ny, nz, seed=seed, nseed=5, continuous=cont, smooth=False,
                        beta=8.0)
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    o = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps, tol=1e-13)
    xb, H, c, edges, w = energy.minimise(g.ravel(), dims, p.fixed[0].ravel(),
                                         p.values[0, 0].ravel(), p.beta, p.eps)
    np.testing.assert_allclose(o["x"].ravel(), xb, atol=1e-9)


@pytest.mark.parametrize("seed", [20, 21, 22])
def test_pcg_equals_dense_direct_8cubed(seed):
    """Oracle Jacobi-PCG to 1e-10 vs numpy.linalg.solve of the same dense L_UU (<= 8^3,
    S:213/S:227).  Pins the CG recurrence and stopping rule."""
    p = wl.random_brick(8, 8, 8, seed=seed, nseed=12, continuous=(seed % 2 == 0), shell=(seed == 22))
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    s = ro.System(g.size, ro.edge_list(g, p.beta, p.eps), p.fixed[0], p.values[0, 0])
    xd = np.linalg.solve(s.L_UU.toarray(), s.b)
    o = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps, tol=1e-10)
    np.testing.assert_allclose(o["x"].ravel()[s.U], xd, atol=1e-9)
    assert o["true_rel"] <= 1e-9


def test_pcg_stopping_rule_and_iteration_count():
    """Iteration count semantics (reading c5): a system already solved takes 0 iterations;
    a looser tol never takes more iterations than a tighter one; absolute mode stops at ||r||<=tol."""
    p = wl.random_brick(8, 8, 8, seed=30, nseed=12)
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    a = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps, tol=1e-4)
    b = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps, tol=1e-10)
    assert 0 < a["iters"] <= b["iters"] and a["rel"] <= 1e-4
    c = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps, tol=1e-10,
                       x0=b["x"].ravel())
    assert c["iters"] <= 1
    d = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps, tol=1e-3, tol_mode=1)
    assert d["rel"] <= 1e-3
    m = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps, tol=1e-12, max_iter=3)
    assert m["iters"] == 3


# ------------------------------------------------------------------ invariants
def test_max_principle_and_seed_invariance():
    """min(values) <= x <= max(values) without clamping; seeds untouched."""
    for seed in range(40, 44):
        p = wl.random_brick(7, 6, 5, seed=seed, nseed=9, continuous=True)
        v = p.values[0, 0][p.fixed[0] > 0]
        g = ro.normalise(p.vol[0], p.scale, p.offset)
        o = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps)
        x = o["x"]
        assert x.min() >= v.min() - 1e-9 and x.max() <= v.max() + 1e-9
        assert np.array_equal(x[p.fixed[0] > 0], p.values[0, 0][p.fixed[0] > 0].astype(np.float64))


def test_mirror_symmetry():
    """Mirroring intensities and seeds along an axis mirrors the solution (S:228 / P:77)."""
    p = wl.random_brick(6, 5, 4, seed=50, nseed=7, continuous=True)
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    o = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps)
    om = ro.solve_brick(g[:, ::-1, :].copy(), p.fixed[0][:, ::-1, :], p.values[0, 0][:, ::-1, :],
                        p.beta, p.eps)
    np.testing.assert_allclose(om["x"], o["x"][:, ::-1, :], atol=1e-9)


def test_energy_decrease():
    """D(x*) <= D(x0) for the default x0 = 0.5 (x* minimises D)."""
    p = wl.random_brick(5, 4, 4, seed=60, nseed=6)
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    o = ro.solve_brick(g, p.fixed[0], p.values[0, 0], p.beta, p.eps)
    edges = energy.grid_edges(5, 4, 4)
    w = energy.weights(list(g.ravel()), edges, p.beta, p.eps)
    x0 = np.where(p.fixed[0].ravel() > 0, p.values[0, 0].ravel(), 0.5)
    assert energy.dirichlet_energy(o["x"].ravel(), edges, w) <= energy.dirichlet_energy(x0, edges, w)


def test_multilabel_sum_to_one_and_argmax():
    """K one-vs-rest probabilities sum to 1 (linearity of the Dirichlet problem);
    argmax picks the class of each seed."""
    rng = np.random.default_rng(70)
    n = 6
    vol = rng.uniform(0, 1, (1, n, n, n)).astype(np.float32)
    labels = np.zeros((1, n, n, n), np.uint8)
    flat = labels.reshape(-1)
    pick = rng.choice(n ** 3, 12, replace=False)
    flat[pick] = np.arange(12) % 4 + 1
    lp = wl.LabelProblem("ml", vol, "f32", labels, 4, beta=10.0)
    o = ro.solve_labels(lp)
    np.testing.assert_allclose(o["x"].sum(axis=0), 1.0, atol=1e-9)
    seeded = labels[0] > 0
    assert np.array_equal(o["labels"][0][seeded], labels[0][seeded])
    # the tie rule is pinned through solve_labels in test_solve_labels_tie_goes_to_lowest_class


def test_degenerate_cases():
    """No fixed voxel -> x0 (0.5), 0 iterations; all fixed -> values; b = 0 -> x_U = 0."""
    g = np.full((2, 2, 4), 0.3)
    o = ro.solve_brick(g, np.zeros(16, int), np.zeros(16), 100.0, 1e-6)
    assert o["iters"] == 0 and np.all(o["x"] == 0.5)
    o = ro.solve_brick(g, np.ones(16, int), np.linspace(0, 1, 16), 100.0, 1e-6)
    np.testing.assert_array_equal(o["x"].ravel(), np.linspace(0, 1, 16))
    f = np.zeros(16, int); f[[0, 5]] = 1
    o = ro.solve_brick(g, f, np.zeros(16), 100.0, 1e-6)
    assert o["iters"] == 0 and np.all(o["x"] == 0.0)


def test_threshold_golden():
    p, m = read_golden("threshold_ramp.txt")
    assert ro.threshold(np.array(p, float)).tolist() == [int(v) for v in m]


def test_normalise_golden():
    """Worked values of reading c2 (tests/golden/normalise.txt) through the per-dtype
    scale / offset the workloads and the ABI use (workloads.NORM)."""
    for dt, v, g in read_golden("normalise.txt"):
        sc, off = gen.NORM[dt]
        raw = np.array([float(v)]).astype(gen.NP_DTYPE[dt])
        assert abs(ro.normalise(raw, sc, off)[0] - float(g)) <= 1e-12, (dt, v, g)


@pytest.mark.parametrize("order", [(1, 2), (2, 1)])
def test_solve_labels_tie_goes_to_lowest_class(order):
    """Reading c11 / S:337 through solve_labels itself: a mirror-symmetric 1 x 1 x 5 chain of
    uniform intensity with a class-a seed at x = 0 and a class-b seed at x = 4.  By symmetry
    both classes' probabilities at the centre are exactly 0.5 (the CG iterates stay
    antisymmetric about it), so the centre voxel takes class 1 whichever end class 1 is
    seeded at; voxels 1 and 3 take the class of their nearer seed."""
    a, b = order
    vol = np.full((1, 1, 1, 5), 0.5, np.float32)
    labels = np.zeros((1, 1, 1, 5), np.uint8)
    labels[0, 0, 0, 0], labels[0, 0, 0, 4] = a, b
    o = ro.solve_labels(wl.LabelProblem("tie", vol, "f32", labels, 2, beta=10.0))
    assert o["prob"][0, 0, 0, 0, 2] == 0.5 and o["prob"][1, 0, 0, 0, 2] == 0.5
    assert o["labels"][0, 0, 0].tolist() == [a, a, 1, b, b]
