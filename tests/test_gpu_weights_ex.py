"""GPU parity of rw_brick_weights_ex (Poisson P:133, Gaussian statistical
model P:127, t-test P:123-125) against oracle/weights_oracle.py, and of solves that use those
weights (streaming and brick-resident solvers) against the fp64 oracle solve."""
import numpy as np
import pytest
import torch

import paper_2103_09564_b200 as rwb
import workloads as wl
from oracle import rw_oracle as ro
from oracle import weights_oracle as wo
from gpu_helpers import dev, assert_prob_parity, assert_label_parity

pytestmark = pytest.mark.gpu

EPS = 1e-6
# fp32 arithmetic on the GPU vs fp64 in the oracle (DESIGN.md §3 R19-R21): sqrt of counts
# up to 2^16 carries ~1.5e-5 absolute error, the exponent/erfc arguments ~1e-6 relative
TOL = {"poisson": (1e-5, 5e-5), "gaussian": (1e-4, 1e-7), "ttest": (2e-4, 2e-6)}


def poisson_volume(nx, ny, nz, batch, seed):
    """Seeded u16 photon counts: background ~3000, a bright blob ~30000 (config-5 levels)."""
    rng = np.random.default_rng([11, seed])
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    lam = np.full((batch, nz, ny, nx), 3000.0)
    for b in range(batch):
        c = rng.uniform(0.3, 0.7, 3) * [nx, ny, nz]
        r = rng.uniform(0.2, 0.3) * min(nx, ny, nz)
        lam[b][(x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 < r * r] = 30000.0
    return np.clip(rng.poisson(lam), 0, 65535).astype(np.uint16)


def oracle_planes(kind, vol, scale, offset, **kw):
    return np.stack([wo.planes(kind, vol[b], scale, offset, EPS, **kw) for b in range(vol.shape[0])], 1)


@pytest.mark.parametrize("kind,dtype", [("poisson", "u16"), ("poisson", "f32"), ("gaussian", "u16"),
                                        ("gaussian", "f32"), ("gaussian", "i16"), ("ttest", "u16"),
                                        ("ttest", "f32"), ("ttest", "u8")])
def test_weights_ex_match_oracle(kind, dtype):
    if kind == "poisson" and dtype == "u16":
        vol = poisson_volume(20, 9, 7, 2, seed=1)
        scale, offset = 1 / 65535, 0.0
    else:
        p = wl.random_brick(20, 9, 7, seed=2, batch=2, dtype=dtype)
        vol, scale, offset = p.vol, p.scale, p.offset
        if kind == "poisson":
            vol = (vol * 500.0).astype(np.float32)      # counts up to 500
    cs = 0.5 if kind == "poisson" else 1.0
    W, dinv = rwb.brick_weights_ex(dev(vol), kind=kind, eps=EPS, count_scale=cs, radius=1,
                                   norm=(scale, offset))
    torch.cuda.synchronize()
    Wo = oracle_planes(kind, vol, scale, offset, count_scale=cs, radius=1)
    rtol, atol = TOL[kind]
    np.testing.assert_allclose(W.cpu().numpy(), Wo, rtol=rtol, atol=atol)
    # dinv from the weights (the Jacobi preconditioner the solvers use)
    s = Wo[0] + Wo[1] + Wo[2]
    s[..., 1:] += Wo[0][..., :-1]
    s[..., 1:, :] += Wo[1][..., :-1, :]
    s[:, 1:] += Wo[2][:, :-1]
    np.testing.assert_allclose(dinv.cpu().numpy(), 1.0 / s, rtol=max(rtol, 1e-5) * 4, atol=atol * 10)


def test_ttest_radius2_and_weight_errors():
    p = wl.random_brick(12, 8, 6, seed=3, dtype="f32")
    W, _ = rwb.brick_weights_ex(dev(p.vol), kind="ttest", eps=EPS, radius=2, norm=(p.scale, p.offset))
    torch.cuda.synchronize()
    Wo = oracle_planes("ttest", p.vol, p.scale, p.offset, radius=2)
    np.testing.assert_allclose(W.cpu().numpy(), Wo, rtol=TOL["ttest"][0], atol=TOL["ttest"][1])
    from paper_2103_09564_b200._lib import RWError
    with pytest.raises(RWError, match="RW_EINVAL"):
        rwb.brick_weights_ex(dev(p.vol), kind="ttest", radius=0)
    with pytest.raises(RWError, match="RW_EINVAL"):
        rwb.brick_weights_ex(dev(p.vol), kind="poisson", count_scale=0.0)


@pytest.mark.parametrize("kind", ["poisson", "gaussian", "ttest"])
@pytest.mark.parametrize("solver", ["streaming", "resident"])
def test_solve_with_alternative_weights(kind, solver):
    """32^3 bricks (the paper's brick size): GPU weights -> GPU solve vs the oracle's
    weights -> fp64 solve; bars of the north star (|dp| <= 1e-4, labels outside 1e-3)."""
    n = 32
    if kind == "poisson":
        vol = poisson_volume(n, n, n, 2, seed=4)
        p = wl.random_brick(n, n, n, seed=5, batch=2, nseed=n ** 3 // 60, continuous=True)
        p.vol, p.dtype, p.scale, p.offset = vol, "u16", 1 / 65535, 0.0
    else:
        p = wl.random_brick(n, n, n, seed=6, batch=2, nseed=n ** 3 // 60, continuous=True, dtype="u16")
    W, _ = rwb.brick_weights_ex(dev(p.vol), kind=kind, eps=EPS, count_scale=1.0,
                                norm=(p.scale, p.offset), want_dinv=False)
    with rwb.solver(solver):
        out = rwb.solve_bricks(dev(p.fixed), dev(p.values), W=W, tol=1e-7, max_iter=20000, labels=True)
    torch.cuda.synchronize()
    prob = out["prob"].cpu().numpy()
    assert (out["status"].cpu().numpy() == 1).all()
    for b in range(2):
        Wo = wo.planes(kind, p.vol[b], p.scale, p.offset, EPS)
        o = ro.solve_brick(np.zeros(p.vol[b].shape), p.fixed[b], p.values[0, b],
                           0.0, EPS, tol=1e-11, edges=wo.planes_to_edges(Wo))
        ref = np.where(p.fixed[b] > 0, p.values[0, b], np.clip(o["x"], 0, 1))
        assert_prob_parity(prob[0, b], ref)
        assert_label_parity(out["labels"].cpu().numpy()[b], ref)
