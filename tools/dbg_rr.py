import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200._lib import lib
import workloads as wl
from oracle import rw_oracle as ro
from test_gpu_fullsize import residual_fp64
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
p = wl.random_brick(48, 40, 36, seed=3, nseed=200, continuous=True)
ref = ro.solve_problem(p, tol=1e-12)
g = ro.normalise(p.vol[0], p.scale, p.offset)
for rr in (0, 4, 16, 64):
    lib().rw_set_option(2, rr)
    with rwb.solver("streaming"):
        o = rwb.solve_bricks(d(p.fixed), d(p.values), vol=d(p.vol), beta=p.beta, eps=p.eps, tol=1e-7, max_iter=5000)
    torch.cuda.synchronize()
    x = o["prob"].cpu().numpy()[0, 0]
    print(json.dumps({"rr": rr, "iters": int(o["iters"][0, 0]), "status": int(o["status"][0, 0]),
                      "resid": float(o["resid"][0, 0]), "true": residual_fp64(g, p.fixed[0], p.values[0, 0], x, p.beta, p.eps),
                      "maxdp": float(np.abs(x - ref["prob"][0, 0]).max())}))
