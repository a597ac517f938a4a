"""cfg2 batch on the resident solver with and without the L2 worker clusters
(RW_OPT_L2_WORKERS): bitwise comparison of every output and timing; RW_L2_RMIN sweep.
    python tools/l2w_ab.py [B] [rmin ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb  # noqa: E402
from paper_2103_09564_b200 import api  # noqa: E402
import workloads as wl  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
rmins = [int(a) for a in sys.argv[2:]] or [48]
p = wl.cfg2(batch=B, workers=16)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
ws = api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, p.dims, 1), "cuda")
res = {}


def run_cfg(on):
    out = {}

    def run():
        with rwb.l2_workers(on):
            out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                        max_iter=p.max_iter, labels=True, workspace=ws))
    run()
    torch.cuda.synchronize()
    api.profile_enable(True)
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    prof = api.profile_read()
    api.profile_enable(False)
    it = out["iters"].cpu().numpy()
    ms = float(np.median(ts))
    o = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    return ms, it, prof, o


ms0, it0, prof0, o0 = run_cfg(False)
print(json.dumps({"workers": 0, "ms": ms0, "G": float(it0.sum()) * 64 ** 3 / ms0 / 1e6,
                  "kernels": {k: v[1] / 5 for k, v in prof0.items() if v[1] > 0}}), flush=True)
for rm in rmins:
    os.environ["RW_L2_RMIN"] = str(rm)
    ms1, it1, prof1, o1 = run_cfg(True)
    same = {k: bool(np.array_equal(o0[k], o1[k])) for k in o0}
    print(json.dumps({"workers": 1, "rmin": rm, "ms": ms1, "G": float(it1.sum()) * 64 ** 3 / ms1 / 1e6,
                      "kernels": {k: v[1] / 5 for k, v in prof1.items() if v[1] > 0},
                      "bitwise_equal": same, "max_dp": float(np.abs(o0["prob"] - o1["prob"]).max())}),
          flush=True)
