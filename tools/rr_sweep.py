"""Residual-replacement interval sweep on cfg3 / cfg4: iterations, time and the fp64 true
residual of the fp32 solution (tests/test_gpu_fullsize.residual_fp64)."""
import os, sys, json, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200._lib import lib
import workloads as wl
from oracle import rw_oracle as ro
from test_gpu_fullsize import residual_fp64

which = sys.argv[1]
rrs = [int(v) for v in sys.argv[2:]]
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
if which == "cfg3":
    p = wl.cfg3()
    g = ro.normalise(p.vol[0], p.scale, p.offset)
    for rr in rrs:
        lib().rw_set_option(2, rr)
        torch.cuda.synchronize(); t = time.time()
        out = rwb.solve_bricks(d(p.fixed), d(p.values), vol=d(p.vol), beta=p.beta, eps=p.eps, tol=p.tol,
                               max_iter=p.max_iter, norm=(p.scale, p.offset))
        torch.cuda.synchronize(); dt = time.time() - t
        x = out["prob"].cpu().numpy()[0, 0]
        rel = residual_fp64(g, p.fixed[0], p.values[0, 0], x, p.beta, p.eps)
        print(json.dumps({"cfg": "cfg3", "rr": rr, "s": dt, "iters": int(out["iters"][0, 0]),
                          "status": int(out["status"][0, 0]), "true_rel_resid": rel}), flush=True)
else:
    lp = wl.cfg4()
    g = ro.normalise(lp.vol[0], lp.scale, lp.offset)
    seeds = lp.labels[0]
    for rr in rrs:
        lib().rw_set_option(2, rr)
        torch.cuda.synchronize(); t = time.time()
        out = rwb.solve_labels(d(lp.labels), lp.K, vol=d(lp.vol), beta=lp.beta, eps=lp.eps, tol=lp.tol,
                               max_iter=lp.max_iter)
        torch.cuda.synchronize(); dt = time.time() - t
        prob = out["prob"].cpu().numpy()[:, 0]
        rels = [residual_fp64(g, seeds > 0, (seeds == k + 1).astype(np.float64), prob[k], lp.beta, lp.eps)
                for k in range(lp.K - 1)]
        print(json.dumps({"cfg": "cfg4", "rr": rr, "s": dt, "iters": out["iters"].cpu().numpy().ravel().tolist(),
                          "true_rel_resid": rels}), flush=True)
