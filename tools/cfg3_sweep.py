"""cfg3 (512x512x256 i16) streaming pass-A rate over a fixed number of iterations, for a list
of z-chunks (RW_OPT_STREAM_ZC) and x-tile widths (RW_TPX).  Usage: cfg3_sweep.py ITERS zc:tpx ..."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200._lib import lib
import workloads as wl

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
combos = sys.argv[2:] or ["0:16", "32:16", "37:16", "43:16", "16:16"]
p = wl.cfg3()
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
fixed, values, vol = d(p.fixed), d(p.values), d(p.vol)
n = int(np.prod(p.dims))
ref = None
for c in combos:
    zc, tpx = (int(v) for v in c.split(":"))
    lib().rw_set_option(6, zc)
    os.environ["RW_TPX"] = str(tpx)
    run = lambda: rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=1e-30,
                                   max_iter=iters)
    with rwb.solver("streaming"):
        o = run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); o = run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    it = int(o["iters"].cpu().numpy().ravel()[0])
    pr = o["prob"].cpu().numpy()
    if ref is None:
        ref = pr
    ms = float(np.median(ts))
    g = n * it / ms / 1e6
    print(json.dumps({"zc": zc, "tpx": tpx, "iters": it, "ms": ms, "G_voxit_s": g,
                      "hbm_frac_38B": g * 38 / 6537.0, "max_dp_vs_first": float(np.abs(pr - ref).max())}),
          flush=True)
lib().rw_set_option(6, 0)
