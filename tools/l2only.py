"""L2 worker clusters in isolation (RW_L2_ONLY=1): cfg2 batch solved by k_l2res alone with
RW_L2_NW worker clusters, timing + bitwise comparison with the default (clusters + workers).
    python tools/l2only.py [B] [nw ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb  # noqa: E402
from paper_2103_09564_b200 import api  # noqa: E402
import workloads as wl  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
nws = [int(a) for a in sys.argv[2:]] or [9]
p = wl.cfg2(batch=B, workers=16)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
ws = api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, p.dims, 1), "cuda")


def run_cfg(reps=3):
    out = {}

    def run():
        out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                    max_iter=p.max_iter, labels=True, workspace=ws))
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    it = out["iters"].cpu().numpy()
    o = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    return float(np.median(ts)), it, o


os.environ.pop("RW_L2_ONLY", None)
ms0, it0, o0 = run_cfg()
print(json.dumps({"mode": "default", "B": B, "ms": ms0, "G": float(it0.sum()) * 64 ** 3 / ms0 / 1e6}), flush=True)
for nw in nws:
    os.environ["RW_L2_ONLY"] = "1"
    os.environ["RW_L2_NW"] = str(nw)
    ms1, it1, o1 = run_cfg(1)
    G = float(it1.sum()) * 64 ** 3 / ms1 / 1e6
    print(json.dumps({"mode": "l2only", "nw": nw, "sms": 4 * nw, "ms": ms1, "G": G, "G_per_sm": G / (4 * nw),
                      "bitwise_equal": {k: bool(np.array_equal(o0[k], o1[k])) for k in o0}}), flush=True)
os.environ.pop("RW_L2_ONLY", None)
