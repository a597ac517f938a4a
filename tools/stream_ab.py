"""Streaming-solver A/B (run once per library via RW_LIB_PATH): cfg3 capped at 300
iterations, the cfg2 batch (512 x 64^3) and cfg4 (256^3, 3 rhs) full solves.  Prints the
median time of 3 runs and a hash of prob / iters per case, so two builds can be compared
bit for bit.    python tools/stream_ab.py [cases: cfg3,cfg2,cfg4]"""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb  # noqa: E402
import workloads as wl  # noqa: E402

cases = (sys.argv[1] if len(sys.argv) > 1 else "cfg3,cfg2,cfg4").split(",")
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()


def h(*arrs):
    m = hashlib.sha1()
    for a in arrs:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:16]


def timed(run):
    out = run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); out = run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return out, float(np.median(ts))


with rwb.solver("streaming"):
    if "cfg3" in cases:
        p = wl.cfg3()
        f, v, vol = d(p.fixed), d(p.values), d(p.vol)
        o, ms = timed(lambda: rwb.solve_bricks(f, v, vol=vol, beta=p.beta, eps=p.eps, tol=1e-30, max_iter=300))
        print(json.dumps({"case": "cfg3_300it", "ms": ms, "hash": h(o["prob"].cpu().numpy(), o["iters"].cpu().numpy())}), flush=True)
        del f, v, vol, o
    if "cfg2" in cases:
        p = wl.cfg2(batch=512, workers=8)
        f, v, vol = d(p.fixed), d(p.values), d(p.vol)
        o, ms = timed(lambda: rwb.solve_bricks(f, v, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol, max_iter=p.max_iter))
        it = o["iters"].cpu().numpy()
        print(json.dumps({"case": "cfg2_stream", "ms": ms, "G_voxit_s": float(it.sum()) * 64 ** 3 / ms / 1e6,
                          "hash": h(o["prob"].cpu().numpy(), it)}), flush=True)
        del f, v, vol, o
    if "cfg4" in cases:
        lp = wl.cfg4()
        lab, vol = d(lp.labels), d(lp.vol)
        o, ms = timed(lambda: rwb.solve_labels(lab, lp.K, vol=vol, beta=lp.beta, eps=lp.eps, tol=lp.tol,
                                               max_iter=lp.max_iter))
        print(json.dumps({"case": "cfg4", "ms": ms, "iters": o["iters"].cpu().numpy().ravel().tolist(),
                          "hash": h(o["prob"].cpu().numpy(), o["iters"].cpu().numpy())}), flush=True)
