"""Brute-force Dirichlet energy and its exact minimiser on tiny bricks (TEST INFRASTRUCTURE).

P:77: the random walker solution minimises D(x) = 1/2 sum_{||p-q||=1} w_pq (x(p)-x(q))^2
subject to the fixed values x(p_m).  This module evaluates D with plain Python loops
over voxels and their +x/+y/+z neighbours (no vectorised slicing, no sparse matrix) and
minimises it by reading the quadratic's Hessian and linear term off point evaluations of
D, then calling ``numpy.linalg.solve``.  It shares no code with rw_oracle.py, so it pins
that module's edge enumeration and Laplacian assembly.
"""
from __future__ import annotations

import math

import numpy as np


def grid_edges(nx, ny, nz):
    """(p, q) voxel index pairs for every 6-neighbour edge, x fastest."""
    out = []
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                p = (z * ny + y) * nx + x
                if x + 1 < nx:
                    out.append((p, p + 1))
                if y + 1 < ny:
                    out.append((p, p + nx))
                if z + 1 < nz:
                    out.append((p, p + nx * ny))
    return out


def weights(gflat, edges, beta, eps):
    return [math.exp(-beta * (gflat[p] - gflat[q]) ** 2) + eps for p, q in edges]


def dirichlet_energy(x, edges, w):
    """D(x) = 1/2 sum_edges w_pq (x_p - x_q)^2."""
    s = 0.0
    for (p, q), wk in zip(edges, w):
        d = x[p] - x[q]
        s += wk * d * d
    return 0.5 * s


def minimise(gflat, dims, fixed, xs, beta, eps):
    """Exact minimiser of D over the unfixed voxels, from point evaluations of D only.

    D restricted to x_U is f(u) = 1/2 u^T H u - c^T u + f0.  With e_i unit vectors:
    f0 = f(0), H_ii = f(e_i) + f(-e_i) - 2 f0, c_i = (f(-e_i) - f(e_i)) / 2,
    H_ij = f(e_i + e_j) - f(e_i) - f(e_j) + f0 for every pair i != j.
    The minimiser solves H u = c.
    """
    nx, ny, nz = dims
    edges = grid_edges(nx, ny, nz)
    w = weights(list(map(float, gflat)), edges, beta, eps)
    fixed = [bool(f) for f in fixed]
    U = [i for i, f in enumerate(fixed) if not f]
    base = [float(xs[i]) if fixed[i] else 0.0 for i in range(len(fixed))]

    def f(assign):
        x = list(base)
        for i, v in assign.items():
            x[i] += v
        return dirichlet_energy(x, edges, w)

    f0 = f({})
    fi = [f({u: 1.0}) for u in U]
    fm = [f({u: -1.0}) for u in U]
    m = len(U)
    H = np.zeros((m, m))
    c = np.zeros(m)
    for a in range(m):
        H[a, a] = fi[a] + fm[a] - 2.0 * f0      # f(+-e_i) = H_ii/2 -+ c_i + f0
        c[a] = (fm[a] - fi[a]) / 2.0
    for a in range(m):                          # every pair, no sparsity assumed
        for b in range(a + 1, m):
            H[a, b] = H[b, a] = f({U[a]: 1.0, U[b]: 1.0}) - fi[a] - fi[b] + f0
    u = np.linalg.solve(H, c) if m else np.zeros(0)
    x = np.array(base)
    x[U] = u
    return x, H, c, edges, w
