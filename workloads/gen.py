"""Seeded synthetic workloads for BASELINE.json configs 1-5 plus the small pin cases.

Recipes follow BASELINE.json ``configs`` and SURVEY.md §8(d) (the readings c2, c3,
c7, c11, c13, c14 are listed in DESIGN.md §3).  Every generator is a pure function
of its arguments (numpy PCG64 ``default_rng`` keyed as documented per function).

Layout convention shared with the C ABI (include/rw.h): arrays are
``[batch, nz, ny, nx]`` (x fastest); per-RHS arrays are ``[nrhs, batch, nz, ny, nx]``.

No edge weight, Laplacian, solver or downsampling arithmetic appears here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

# ABI dtype names and the normalisation that maps them onto [0, 1] (reading c2).
NORM = {
    "u8": (1.0 / 255.0, 0.0),
    "u16": (1.0 / 65535.0, 0.0),
    "i16": (1.0 / 2000.0, 0.5),     # HU window [-1000, 1000] -> (v + 1000) / 2000
    "f32": (1.0, 0.0),
}
NP_DTYPE = {"u8": np.uint8, "u16": np.uint16, "i16": np.int16, "f32": np.float32}


@dataclass
class Problem:
    """One batched solve: ``rw_solve_bricks`` inputs."""
    name: str
    vol: np.ndarray                 # [B, nz, ny, nx], dtype per ``dtype``
    dtype: str                      # 'u8' | 'u16' | 'i16' | 'f32'
    fixed: np.ndarray               # uint8 [B, nz, ny, nx]; 1 = Dirichlet voxel
    values: np.ndarray              # float32 [R, B, nz, ny, nx]; read only where fixed
    beta: float = 100.0
    eps: float = 1e-6
    tol: float = 1e-6
    max_iter: int = 5000
    tol_mode: int = 0               # 0 relative ||r||/||b||, 1 absolute ||r||
    scale: float = field(default=None)
    offset: float = field(default=None)

    def __post_init__(self):
        if self.scale is None:
            self.scale, self.offset = NORM[self.dtype]

    @property
    def batch(self):
        return self.vol.shape[0]

    @property
    def dims(self):                 # (nx, ny, nz)
        B, nz, ny, nx = self.vol.shape
        return nx, ny, nz

    @property
    def nrhs(self):
        return self.values.shape[0]

    def subset(self, idx):
        idx = list(idx)
        return Problem(self.name + f"[{len(idx)}]", self.vol[idx].copy(), self.dtype,
                       self.fixed[idx].copy(), self.values[:, idx].copy(), self.beta,
                       self.eps, self.tol, self.max_iter, self.tol_mode, self.scale,
                       self.offset)


@dataclass
class LabelProblem:
    """One multi-label solve: ``rw_solve_labels`` inputs (classes 1..K, 0 = unseeded)."""
    name: str
    vol: np.ndarray
    dtype: str
    labels: np.ndarray              # uint8 [B, nz, ny, nx]
    K: int
    beta: float = 100.0
    eps: float = 1e-6
    tol: float = 1e-6
    max_iter: int = 5000
    scale: float = field(default=None)
    offset: float = field(default=None)

    def __post_init__(self):
        if self.scale is None:
            self.scale, self.offset = NORM[self.dtype]

    @property
    def dims(self):
        B, nz, ny, nx = self.vol.shape
        return nx, ny, nz


def _centres(nx, ny, nz):
    """Voxel-centre coordinates (x+0.5, y+0.5, z+0.5) broadcastable over [nz, ny, nx]."""
    z = (np.arange(nz, dtype=np.float64) + 0.5)[:, None, None]
    y = (np.arange(ny, dtype=np.float64) + 0.5)[None, :, None]
    x = (np.arange(nx, dtype=np.float64) + 0.5)[None, None, :]
    return x, y, z


def _ellipsoid(x, y, z, c, a):
    return ((x - c[0]) / a[0]) ** 2 + ((y - c[1]) / a[1]) ** 2 + ((z - c[2]) / a[2]) ** 2 <= 1.0


# --------------------------------------------------------------------------- config 1
def cfg1() -> Problem:
    """BASELINE.json configs[0]: single 32^3 fp32 brick, seed 0 (reading c14).

    Sphere radius 10 centred at (16,16,16) (voxel centres at i+0.5) at 0.8 on 0.2,
    + N(0, 0.05), clamp [0,1]; 20 fg seeds uniformly without replacement among voxels
    at distance <= 6; 20 bg seeds among voxels whose every coordinate is in
    [0,4) U [28,32).  RNG draw order: noise, fg seeds, bg seeds.  No Dirichlet faces.
    """
    n = 32
    rng = np.random.default_rng(0)
    x, y, z = _centres(n, n, n)
    d = np.sqrt((x - 16) ** 2 + (y - 16) ** 2 + (z - 16) ** 2)
    g = np.where(d <= 10.0, 0.8, 0.2)
    g = g + rng.normal(0.0, 0.05, size=(n, n, n))
    g = np.clip(g, 0.0, 1.0).astype(np.float32)
    fg_c = np.flatnonzero((d <= 6.0).ravel())
    fg = rng.choice(fg_c, 20, replace=False)
    i = np.arange(n)
    corner = (i < 4) | (i >= n - 4)
    cm = corner[None, None, :] & corner[None, :, None] & corner[:, None, None]
    bg_c = np.flatnonzero(cm.ravel())
    bg = rng.choice(bg_c, 20, replace=False)
    fixed = np.zeros(n ** 3, np.uint8)
    values = np.zeros(n ** 3, np.float32)
    fixed[fg] = 1
    values[fg] = 1.0
    fixed[bg] = 1
    values[bg] = 0.0
    return Problem("cfg1", g.reshape(1, n, n, n), "f32", fixed.reshape(1, n, n, n),
                   values.reshape(1, 1, n, n, n), beta=100.0, eps=1e-6, tol=1e-6,
                   max_iter=5000)


# --------------------------------------------------------------------------- config 2
def _trilinear_lattice(lat, n):
    """Trilinear interpolation of a 5^3 lattice (corners at 0 and n) onto voxel centres."""
    m = lat.shape[0] - 1
    t = (np.arange(n) + 0.5) / n * m
    i0 = np.minimum(np.floor(t).astype(int), m - 1)
    f = t - i0
    # separable: interpolate along x, then y, then z
    a = lat[:, :, i0] * (1 - f)[None, None, :] + lat[:, :, i0 + 1] * f[None, None, :]
    a = a[:, i0, :] * (1 - f)[None, :, None] + a[:, i0 + 1, :] * f[None, :, None]
    a = a[i0, :, :] * (1 - f)[:, None, None] + a[i0 + 1, :, :] * f[:, None, None]
    return a


def cfg2_brick(b: int, n: int = 64, seed_frac: float = 1e-3):
    """One brick of BASELINE.json configs[1], keyed by ``default_rng([1, b])``.

    Background ~U(0.05,0.3); 1-5 ellipsoids with centres U(10,54)^3 and semi-axes
    U(4,14)^3 (scaled by n/64), intensity ~U(0.5,0.9); + N(0,0.03); clamp; quantise
    round(g*65535) to u16.  The one-voxel shell is Dirichlet (reading c3) with values
    from a trilinearly upsampled 5^3 U(0,1) lattice (smooth, in [0,1]).  Seeds:
    round(seed_frac*n^3) split fg/bg; fg inside blobs with >= 1 per blob (reading c7),
    bg outside all blobs; all seeds interior.
    Returns (vol u16 [n,n,n], fixed u8, values f32).
    """
    rng = np.random.default_rng([1, b])
    s = n / 64.0
    bgv = rng.uniform(0.05, 0.3)
    nblob = int(rng.integers(1, 6))
    blobs = []
    for _ in range(nblob):
        c = rng.uniform(10 * s, 54 * s, 3)
        a = rng.uniform(4 * s, 14 * s, 3)
        v = rng.uniform(0.5, 0.9)
        blobs.append((c, a, v))
    x, y, z = _centres(n, n, n)
    g = np.full((n, n, n), bgv)
    masks = []
    for c, a, v in blobs:
        m = _ellipsoid(x, y, z, c, a)
        g[m] = v
        masks.append(m)
    g = g + rng.normal(0.0, 0.03, size=(n, n, n))
    g = np.clip(g, 0.0, 1.0)
    vol = np.rint(g * 65535.0).astype(np.uint16)
    lat = rng.uniform(0.0, 1.0, (5, 5, 5))
    face = _trilinear_lattice(lat, n)
    i = np.arange(n)
    e = (i == 0) | (i == n - 1)
    shell = e[None, None, :] | e[None, :, None] | e[:, None, None]
    interior = ~shell
    nseed = max(2, int(round(seed_frac * n ** 3)))
    nfg = max(nseed // 2, nblob)
    nbg = max(nseed - nseed // 2, 1)
    taken = np.zeros((n, n, n), bool)
    fg = []
    for m in masks:
        cand = np.flatnonzero((m & interior & ~taken).ravel())
        if cand.size:
            k = int(rng.choice(cand))
            fg.append(k)
            taken.flat[k] = True
    union = np.zeros((n, n, n), bool)
    for m in masks:
        union |= m
    cand = np.flatnonzero((union & interior & ~taken).ravel())
    rest = rng.choice(cand, min(nfg - len(fg), cand.size), replace=False)
    fg.extend(int(k) for k in rest)
    taken.flat[rest] = True
    cand = np.flatnonzero((~union & interior).ravel())
    bg = rng.choice(cand, min(nbg, cand.size), replace=False)
    fixed = shell.astype(np.uint8).ravel()
    values = np.where(shell, face, 0.0).astype(np.float32).ravel()
    fixed[fg] = 1
    values[fg] = 1.0
    fixed[bg] = 1
    values[bg] = 0.0
    # reading c7 / R7: every region the intensity contrast isolates must hold a fixed voxel.
    # Union of overlapping ellipsoids can enclose a small background pocket, and a later blob
    # can cut an earlier one in two; such a region would be coupled to the rest only through
    # edges with |dg| > GAP (weights below ~1e-4 at beta = 100), and its solution would stay
    # at the initial guess at tol 1e-6 (unpinned).  One seed goes into each
    # such region: value 1 if its mean intensity is blob-like, else 0.
    _seed_isolated(vol.astype(np.float64) / 65535.0, fixed, values, bgv, n)
    return vol, fixed.reshape(n, n, n), values.reshape(n, n, n)


GAP = 0.3   # intensity jump that separates regions (input conditioning, see _seed_isolated)


def _seed_isolated(g, fixed, values, bgv, n):
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    idx = np.arange(n ** 3).reshape(n, n, n)
    rows, cols = [], []
    for sp, sq in (((slice(None), slice(None), slice(0, -1)), (slice(None), slice(None), slice(1, None))),
                   ((slice(None), slice(0, -1), slice(None)), (slice(None), slice(1, None), slice(None))),
                   ((slice(0, -1), slice(None), slice(None)), (slice(1, None), slice(None), slice(None)))):
        close = np.abs(g[sp] - g[sq]) <= GAP
        rows.append(idx[sp][close])
        cols.append(idx[sq][close])
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    A = coo_matrix((np.ones(r.size, np.int8), (r, c)), shape=(n ** 3, n ** 3))
    ncomp, lab = connected_components(A, directed=False)
    has_fixed = np.zeros(ncomp, bool)
    has_fixed[lab[fixed > 0]] = True
    gr = g.ravel()
    for comp in np.flatnonzero(~has_fixed):
        members = np.flatnonzero(lab == comp)
        k = int(members[0])
        fixed[k] = 1
        values[k] = 1.0 if gr[members].mean() > bgv + 0.15 else 0.0


def cfg2(batch: int = 512, n: int = 64, bricks=None, max_iter: int = 2000,
         workers: int = 0) -> Problem:
    """BASELINE.json configs[1]: ``batch`` independent u16 bricks (brick b keyed [1, b]).

    ``bricks`` selects explicit brick ids (e.g. a sample of the 512) instead of 0..batch-1.
    """
    ids = list(range(batch)) if bricks is None else list(bricks)
    B = len(ids)
    vol = np.empty((B, n, n, n), np.uint16)
    fixed = np.empty((B, n, n, n), np.uint8)
    values = np.empty((1, B, n, n, n), np.float32)
    if workers and B > 8:
        from concurrent.futures import ProcessPoolExecutor
        with ProcessPoolExecutor(workers) as ex:
            outs = ex.map(cfg2_brick, ids, [n] * B, chunksize=max(1, B // (4 * workers)))
            for j, (v, f, val) in enumerate(outs):
                vol[j], fixed[j], values[0, j] = v, f, val
    else:
        for j, b in enumerate(ids):
            vol[j], fixed[j], values[0, j] = cfg2_brick(b, n)
    return Problem(f"cfg2_{B}x{n}^3", vol, "u16", fixed, values, beta=100.0, eps=1e-6,
                   tol=1e-6, max_iter=max_iter)


# --------------------------------------------------------------------------- config 3
# CT-like phantom geometry in normalised coordinates (u = (x+0.5)/nx, ...).
_CT_REGIONS = [
    # (name, centre, semi-axes, HU or None for U(400,1000) bone)
    ("fat", (0.50, 0.50, 0.50), (0.42, 0.32, 0.47), -100.0),
    ("soft", (0.50, 0.50, 0.50), (0.36, 0.26, 0.44), 40.0),
    ("liver", (0.37, 0.45, 0.55), (0.14, 0.12, 0.18), 60.0),
    ("spine", (0.50, 0.72, 0.50), (0.05, 0.05, 0.45), None),
    ("bone2", (0.76, 0.50, 0.30), (0.04, 0.14, 0.08), None),
    ("bone3", (0.24, 0.52, 0.75), (0.04, 0.12, 0.10), None),
]


def cfg3(scale: float = 1.0, seeds_per_region: int = 200, max_iter: int = 20000) -> Problem:
    """BASELINE.json configs[2]: one 512x512x256 int16 CT-like phantom (scale 1).

    Air -1000; nested ellipsoids fat -100, soft tissue 40, liver 60, spine and two more
    bones at HU ~U(400,1000); + N(0, 20) HU, rounded to int16; window [-1000,1000].
    ``seeds_per_region`` seeds inside each of the 7 regions; liver seeds = 1, others 0.
    ``scale`` shrinks every axis (0.25 -> 128x128x64) for parity tests.
    """
    nx, ny, nz = (max(4, int(round(512 * scale)) // 4 * 4), max(2, int(round(512 * scale))),
                  max(2, int(round(256 * scale))))
    rng = np.random.default_rng(3)
    bone_hu = rng.uniform(400.0, 1000.0, 3)
    x, y, z = _centres(nx, ny, nz)
    u, v, w = x / nx, y / ny, z / nz
    region = np.zeros((nz, ny, nx), np.uint8)          # 0 = air
    hu = np.full((nz, ny, nx), -1000.0, np.float32)
    bi = 0
    for k, (name, c, a, h) in enumerate(_CT_REGIONS):
        m = _ellipsoid(u, v, w, c, a)
        if h is None:
            h = bone_hu[bi]
            bi += 1
        hu[m] = h
        region[m] = k + 1
    hu += rng.normal(0.0, 20.0, size=hu.shape).astype(np.float32)
    vol = np.clip(np.rint(hu), -32768, 32767).astype(np.int16)
    fixed = np.zeros(region.size, np.uint8)
    values = np.zeros(region.size, np.float32)
    flat = region.ravel()
    for k in range(len(_CT_REGIONS) + 1):
        cand = np.flatnonzero(flat == k)
        pick = rng.choice(cand, min(seeds_per_region, cand.size), replace=False)
        fixed[pick] = 1
        values[pick] = 1.0 if k == 3 else 0.0           # region 3 = liver
    shp = (1, nz, ny, nx)
    return Problem(f"cfg3_{nx}x{ny}x{nz}", vol.reshape(shp), "i16", fixed.reshape(shp),
                   values.reshape((1,) + shp), beta=100.0, eps=1e-6, tol=1e-6,
                   max_iter=max_iter)


# --------------------------------------------------------------------------- config 4
_ML_BLOBS = [  # class id, centre, semi-axes (normalised), mean
    (1, (0.30, 0.30, 0.50), (0.18, 0.15, 0.30), 0.40),
    (2, (0.70, 0.30, 0.50), (0.15, 0.18, 0.25), 0.65),
    (3, (0.50, 0.72, 0.50), (0.30, 0.15, 0.20), 0.90),
]


def cfg4(n: int = 256, seeds_per_label: int = 100, max_iter: int = 5000) -> LabelProblem:
    """BASELINE.json configs[3]: K = 4 multi-label 256^3 fp32 (reading c11, c13).

    Classes 1..3 are three non-overlapping ellipsoids with means 0.4/0.65/0.9; class 4
    is the background with mean 0.15.  g ~ N(mu_k, 0.04) (sigma = std), clamp [0,1].
    ``seeds_per_label`` seeds per class inside its region.  Class 4 (background) is the
    one derived as 1 - sum by the K-1 RHS solve.
    """
    rng = np.random.default_rng(4)
    x, y, z = _centres(n, n, n)
    u, v, w = x / n, y / n, z / n
    cls = np.full((n, n, n), 4, np.uint8)
    mu = np.full((n, n, n), 0.15)
    for k, c, a, m in _ML_BLOBS:
        msk = _ellipsoid(u, v, w, c, a)
        cls[msk] = k
        mu[msk] = m
    g = np.clip(mu + rng.normal(0.0, 0.04, size=mu.shape), 0.0, 1.0).astype(np.float32)
    labels = np.zeros(n ** 3, np.uint8)
    flat = cls.ravel()
    for k in (1, 2, 3, 4):
        cand = np.flatnonzero(flat == k)
        pick = rng.choice(cand, min(seeds_per_label, cand.size), replace=False)
        labels[pick] = k
    return LabelProblem(f"cfg4_{n}^3", g.reshape(1, n, n, n), "f32",
                        labels.reshape(1, n, n, n), 4, beta=100.0, eps=1e-6, tol=1e-6,
                        max_iter=max_iter)


# --------------------------------------------------------------------------- config 5
def cfg5_dims(scale: float = 1.0):
    d = max(8, int(round(2048 * scale)))
    return d, d, d


def _vessel_segments(d, seed=5, n_trees=None):
    """Random branching vessel trees (SPEC S:406-414 reading): segment length 5r, children
    r/sqrt(2) (area preserving), directions within a 40 deg cone; radius 2..12 voxels at
    full scale; roots start on the volume border pointing inward."""
    rng = np.random.default_rng([5, 0])
    s = d / 2048.0
    rmin, rmax = max(1.0, 2.0 * s), max(1.5, 12.0 * s)
    n_trees = n_trees or 48
    segs = []
    for _ in range(n_trees):
        face = rng.integers(0, 6)
        p = rng.uniform(0, d, 3)
        p[face // 2] = 0.0 if face % 2 == 0 else d
        dirn = np.zeros(3)
        dirn[face // 2] = 1.0 if face % 2 == 0 else -1.0
        stack = [(p, dirn, rng.uniform(0.66 * rmax, rmax), 0)]
        while stack and len(segs) < 20000:
            p0, dv, r, depth = stack.pop()
            p1 = p0 + dv * 5.0 * r
            segs.append((p0, p1, r))
            if r / math.sqrt(2.0) < rmin or depth > 14 or np.any(p1 < 0) or np.any(p1 > d):
                continue
            for _c in range(2):
                # direction within a 40 degree cone around dv
                t = rng.normal(size=3)
                t -= t.dot(dv) * dv
                t /= np.linalg.norm(t) + 1e-12
                ang = math.radians(40.0) * math.sqrt(rng.uniform())
                nd = math.cos(ang) * dv + math.sin(ang) * t
                stack.append((p1, nd / np.linalg.norm(nd), r / math.sqrt(2.0), depth + 1))
    return segs


def cfg5_slab(z0: int, z1: int, scale: float = 1.0, _segs_cache={}):
    """Planes [z0, z1) of the config-5 vessel volume (u16, [z1-z0, d, d]).

    Vessel voxels ~N(30000, sqrt(30000)), background ~N(3000, sqrt(3000)) (Gaussian
    approximation of Poisson), clamp [0, 65535]; noise keyed per plane by
    default_rng([5, 1, z]) so any slab decomposition gives identical volumes.
    """
    d = cfg5_dims(scale)[0]
    if d not in _segs_cache:
        _segs_cache[d] = _vessel_segments(d)
    segs = _segs_cache[d]
    out = np.empty((z1 - z0, d, d), np.uint16)
    yy = (np.arange(d) + 0.5)[:, None]
    xx = (np.arange(d) + 0.5)[None, :]
    for zi, zpl in enumerate(range(z0, z1)):
        zc = zpl + 0.5
        inside = np.zeros((d, d), bool)
        for p0, p1, r in segs:
            lo = min(p0[2], p1[2]) - r
            hi = max(p0[2], p1[2]) + r
            if zc < lo or zc > hi:
                continue
            x0 = int(max(0, math.floor(min(p0[0], p1[0]) - r)))
            x1 = int(min(d, math.ceil(max(p0[0], p1[0]) + r) + 1))
            y0 = int(max(0, math.floor(min(p0[1], p1[1]) - r)))
            y1 = int(min(d, math.ceil(max(p0[1], p1[1]) + r) + 1))
            if x0 >= x1 or y0 >= y1:
                continue
            px, py = xx[:, x0:x1], yy[y0:y1, :]
            ab = p1 - p0
            L2 = ab.dot(ab)
            t = ((px - p0[0]) * ab[0] + (py - p0[1]) * ab[1] + (zc - p0[2]) * ab[2]) / L2
            t = np.clip(t, 0.0, 1.0)
            dx = px - (p0[0] + t * ab[0])
            dy = py - (p0[1] + t * ab[1])
            dz = zc - (p0[2] + t * ab[2])
            inside[y0:y1, x0:x1] |= dx * dx + dy * dy + dz * dz <= r * r
        rng = np.random.default_rng([5, 1, zpl])
        noise = rng.standard_normal((d, d))
        val = np.where(inside, 30000.0 + math.sqrt(30000.0) * noise,
                       3000.0 + math.sqrt(3000.0) * noise)
        out[zi] = np.clip(np.rint(val), 0, 65535).astype(np.uint16)
    return out


# --------------------------------------------------------------------------- small pins
def chain(n: int, g=None, v0: float = 1.0, v1: float = 0.0, dtype="f32") -> Problem:
    """n x 1 x 1 chain with end voxels fixed to v0 / v1."""
    g = np.full(n, 0.5, np.float32) if g is None else np.asarray(g, np.float32)
    fixed = np.zeros(n, np.uint8)
    values = np.zeros(n, np.float32)
    fixed[[0, n - 1]] = 1
    values[0], values[n - 1] = v0, v1
    return Problem(f"chain{n}", g.reshape(1, 1, 1, n), dtype, fixed.reshape(1, 1, 1, n),
                   values.reshape(1, 1, 1, 1, n), beta=100.0, eps=1e-6, tol=1e-10,
                   max_iter=100000)


def layered(nx: int, ny: int, nz: int, seed: int = 0, beta: float = 100.0) -> Problem:
    """g depends on x only (random per plane); plane x=0 fixed 1, plane x=nx-1 fixed 0."""
    rng = np.random.default_rng([7, seed])
    gx = rng.uniform(0.0, 1.0, nx).astype(np.float32)
    g = np.broadcast_to(gx[None, None, :], (nz, ny, nx)).copy()
    fixed = np.zeros((nz, ny, nx), np.uint8)
    values = np.zeros((nz, ny, nx), np.float32)
    fixed[:, :, 0] = 1
    fixed[:, :, -1] = 1
    values[:, :, 0] = 1.0
    return Problem(f"layered{nx}x{ny}x{nz}", g[None], "f32", fixed[None], values[None, None],
                   beta=beta, eps=1e-6, tol=1e-10, max_iter=100000)


def random_brick(nx: int, ny: int, nz: int, seed: int, batch: int = 1, nseed: int = 8,
                 continuous: bool = False, shell: bool = False, nrhs: int = 1,
                 dtype: str = "f32", beta: float = 100.0, smooth: bool = True) -> Problem:
    """Random small bricks for dense-direct pins and parity (keyed default_rng([9, seed])).

    Intensities are a piecewise-constant random pattern plus noise (``smooth``) or i.i.d.
    uniform; ``nseed`` random seed voxels with values in {0,1} (or U(0,1) when
    ``continuous``); optional Dirichlet shell with U(0,1) values.
    """
    rng = np.random.default_rng([9, seed])
    shp = (batch, nz, ny, nx)
    if smooth:
        base = rng.uniform(0, 1, (batch, 2, 2, 2))
        zi = (np.arange(nz) * 2 // max(nz, 1))
        yi = (np.arange(ny) * 2 // max(ny, 1))
        xi = (np.arange(nx) * 2 // max(nx, 1))
        g = base[:, zi][:, :, yi][:, :, :, xi] + rng.normal(0, 0.05, shp)
    else:
        g = rng.uniform(0, 1, shp)
    g = np.clip(g, 0, 1)
    if dtype == "f32":
        vol = g.astype(np.float32)
    elif dtype == "u16":
        vol = np.rint(g * 65535).astype(np.uint16)
    elif dtype == "u8":
        vol = np.rint(g * 255).astype(np.uint8)
    elif dtype == "i16":
        vol = np.rint(g * 2000 - 1000).astype(np.int16)
    else:
        raise ValueError(dtype)
    n = nx * ny * nz
    fixed = np.zeros((batch, n), np.uint8)
    values = np.zeros((nrhs, batch, n), np.float32)
    for b in range(batch):
        k = min(nseed, n)
        pick = rng.choice(n, k, replace=False)
        fixed[b, pick] = 1
        for r in range(nrhs):
            values[r, b, pick] = (rng.uniform(0, 1, k) if continuous
                                  else rng.integers(0, 2, k).astype(np.float32))
    fixed = fixed.reshape(shp)
    values = values.reshape((nrhs,) + shp)
    if shell:
        e = lambda m: (np.arange(m) == 0) | (np.arange(m) == m - 1)
        sh = e(nx)[None, None, :] | e(ny)[None, :, None] | e(nz)[:, None, None]
        sv = rng.uniform(0, 1, (nrhs,) + shp).astype(np.float32)
        fixed = np.where(sh[None], 1, fixed).astype(np.uint8)
        values = np.where(sh[None, None], sv, values).astype(np.float32)
    return Problem(f"rand{nx}x{ny}x{nz}s{seed}", vol, dtype, fixed, values, beta=beta,
                   eps=1e-6, tol=1e-10, max_iter=100000)


def pyramid_volume(nx: int, ny: int, nz: int, dtype: str, seed: int, kind: str = "random"):
    """Volumes for the pyramid pins/parity (keyed default_rng([11, seed]))."""
    rng = np.random.default_rng([11, seed])
    dt = NP_DTYPE[dtype]
    shp = (nz, ny, nx)
    if kind == "random":
        if dtype == "f32":
            return rng.uniform(0, 1, shp).astype(np.float32)
        info = np.iinfo(dt)
        return rng.integers(info.min, int(info.max) + 1, shp, dtype=np.int64).astype(dt)
    if kind == "max":
        return np.full(shp, np.iinfo(dt).max if dtype != "f32" else 1.0, dt)
    if kind == "min":
        return np.full(shp, np.iinfo(dt).min if dtype != "f32" else 0.0, dt)
    raise ValueError(kind)


def cfg5_volume(scale: float = 1.0, workers: int = 16):
    """The whole config-5 vessel volume [d, d, d] u16 (cfg5_slab over z-slabs on `workers`
    host threads)."""
    from concurrent.futures import ThreadPoolExecutor
    d = cfg5_dims(scale)[0]
    cfg5_slab(0, 1, scale)          # build the segment cache once
    step = max(1, d // (max(1, workers) * 4))
    with ThreadPoolExecutor(max(1, workers)) as ex:
        parts = list(ex.map(lambda z: cfg5_slab(z, min(z + step, d), scale), range(0, d, step)))
    return np.concatenate(parts, 0)


def cfg5_seeds(vol, nfg: int = 400, nbg: int = 400, seed: int = 0):
    """Config 5's rasterised seeds (reading R22): 0 unseeded, 1 foreground at vessel
    segment mid points, 2 background at random voxels whose 5^3 neighbourhood is vessel-free
    (intensity well below the vessel level)."""
    d = vol.shape[0]
    rng = np.random.default_rng([5, 2, seed])
    seeds = np.zeros(vol.shape, np.uint8)
    segs = _vessel_segments(d)
    pick = rng.choice(len(segs), size=min(nfg, len(segs)), replace=False)
    for i in pick:
        p0, p1, r = segs[i]
        m = np.floor((p0 + p1) / 2).astype(int)
        x, y, z = np.clip(m, 0, d - 1)
        if vol[z, y, x] > 15000:
            seeds[z, y, x] = 1
    n = 0
    while n < nbg:
        z, y, x = rng.integers(2, d - 2, 3)
        if vol[z - 2:z + 3, y - 2:y + 3, x - 2:x + 3].max() < 10000:
            seeds[z, y, x] = 2
            n += 1
    return seeds


def cfg5_new_seeds(vol, seeds, n: int = 50, seed: int = 1):
    """Config 5's incremental step: `n` new foreground seeds at vessel segment mid points
    that were not seeded before."""
    d = vol.shape[0]
    rng = np.random.default_rng([5, 3, seed])
    out = seeds.copy()
    segs = _vessel_segments(d)
    added = 0
    for i in rng.permutation(len(segs)):
        p0, p1, r = segs[i]
        x, y, z = np.clip(np.floor((p0 + p1) / 2).astype(int), 0, d - 1)
        if vol[z, y, x] > 15000 and out[z, y, x] == 0:
            out[z, y, x] = 1
            added += 1
            if added == n:
                break
    return out
