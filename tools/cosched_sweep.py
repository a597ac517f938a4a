"""Sweep RW_OPT_COSCHED (streaming share next to the resident clusters) on the cfg2 batch."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200 import api
from paper_2103_09564_b200._lib import lib
import workloads as wl

p = wl.cfg2(batch=512)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
ws = api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, p.dims, 1), "cuda")
ref = None
for pm in [int(x) for x in (sys.argv[1:] or ["0", "120", "160", "200", "240"])]:
    lib().rw_set_option(1, pm)
    out = {}
    def run():
        out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                    max_iter=p.max_iter, workspace=ws))
    run(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    it = out["iters"].cpu().numpy()
    prob = out["prob"].cpu().numpy()
    if ref is None:
        ref = prob
    ms = float(np.median(ts))
    print(json.dumps({"cosched_pm": pm, "ms": ms, "G_voxit_s": float(it.sum()) * 64 ** 3 / ms / 1e6,
                      "status_ok": bool((out["status"].cpu().numpy() == 1).all()),
                      "max_abs_dprob_vs_first": float(np.abs(prob - ref).max())}), flush=True)
