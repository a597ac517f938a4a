"""Resident solver on `batch` cfg2-style bricks of side n (default 40 = the paper's s_e):
time (CUDA events), G voxel-iter/s; RES_DUMP=path.npz keeps prob/iters for A/B."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
import workloads as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
p = wl.cfg2(batch=B, n=n)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
out = {}
def run():
    with rwb.solver("resident"):
        out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                    max_iter=p.max_iter))
run(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    run()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
it = out["iters"].cpu().numpy()
print(json.dumps({"n": n, "batch": B, "ms": ms, "G_voxit_s": float(it.sum()) * n ** 3 / ms / 1e6,
                  "iters": [int(it.min()), float(np.median(it)), int(it.max())]}))
if os.environ.get("RES_DUMP"):
    np.savez(os.environ["RES_DUMP"], prob=out["prob"].cpu().numpy(), it=it)
