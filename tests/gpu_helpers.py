"""Shared helpers of the GPU parity tests: move a workloads.Problem to the device, call the
C ABI through the binding, compare with the oracle using the north-star bars."""
import numpy as np
import torch

import paper_2103_09564_b200 as rwb
from workloads.gen import NP_DTYPE

TORCH_DT = {"u8": torch.uint8, "u16": torch.uint16, "i16": torch.int16, "f32": torch.float32}

# north star (BASELINE.json): |dp| <= 1e-4; labels exact where |p_oracle - 0.5| > 1e-3
P_TOL = 1e-4
LABEL_BAND = 1e-3


def dev(a, dt=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.cuda() if dt is None else t.to(dt).cuda()


def gpu_solve(p, labels=True, x0=None, tol=None, max_iter=None, tol_mode=None, use_W=False,
              **kw):
    vol = dev(p.vol)
    fixed = dev(p.fixed)
    values = dev(p.values)
    W = None
    if use_W:
        W, _ = rwb.brick_weights(vol, beta=p.beta, eps=p.eps, norm=(p.scale, p.offset),
                                 want_dinv=False)
        vol = None
    out = rwb.solve_bricks(fixed, values, vol=vol, W=W, beta=p.beta, eps=p.eps,
                           tol=p.tol if tol is None else tol,
                           max_iter=p.max_iter if max_iter is None else max_iter,
                           tol_mode=p.tol_mode if tol_mode is None else tol_mode,
                           x0=None if x0 is None else dev(x0), norm=(p.scale, p.offset),
                           labels=labels, **kw)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


def assert_prob_parity(gpu_prob, oracle_prob, tol=P_TOL):
    d = np.abs(gpu_prob.astype(np.float64) - oracle_prob)
    assert d.max() <= tol, f"max |dp| = {d.max():.3e} > {tol}"
    return d.max()


def assert_label_parity(gpu_labels, oracle_prob, band=LABEL_BAND):
    sure = np.abs(oracle_prob - 0.5) > band
    want = (oracle_prob > 0.5).astype(np.uint8)
    bad = (gpu_labels != want) & sure
    assert not bad.any(), f"{bad.sum()} label mismatches outside the {band} band"
