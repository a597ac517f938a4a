"""cfg3 / cfg4 streaming solves: time + a hash of the outputs (for bitwise A/B of builds or of
RW_LASTDEC_MIN_U settings run in separate processes).   python tools/lastdec_ab.py TAG"""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb  # noqa: E402
from paper_2103_09564_b200 import api  # noqa: E402
import workloads as wl  # noqa: E402
from tools.bench_configs import ev_time, dev  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "run"


def h(*ts):
    m = hashlib.sha256()
    for t in ts:
        m.update(t.contiguous().cpu().numpy().tobytes())
    return m.hexdigest()[:16]


p = wl.cfg3()
vol, fixed, values = dev(p.vol), dev(p.fixed), dev(p.values)
ws = api.alloc_workspace(rwb.solve_workspace_bytes(1, p.dims, 1), "cuda")
out = {}


def run3():
    out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                max_iter=p.max_iter, workspace=ws))
ms = ev_time(run3, reps=2)
print(json.dumps({"tag": tag, "cfg": "cfg3", "ms": ms, "iters": int(out["iters"].max()),
                  "hash": h(out["prob"], out["iters"], out["resid"])}), flush=True)
del ws, vol, fixed, values
lp = wl.cfg4(n=256)
seeds, vol = dev(lp.labels), dev(lp.vol)
ws = api.alloc_workspace(rwb.solve_labels_workspace_bytes(1, lp.dims, lp.K), "cuda")
out = {}


def run4():
    out.update(rwb.solve_labels(seeds, lp.K, vol=vol, beta=lp.beta, eps=lp.eps, tol=lp.tol,
                                max_iter=lp.max_iter, workspace=ws))
ms = ev_time(run4, reps=2)
print(json.dumps({"tag": tag, "cfg": "cfg4", "ms": ms, "iters": out["iters"].cpu().numpy().ravel().tolist(),
                  "hash": h(out["prob"], out["labels"], out["iters"])}), flush=True)
