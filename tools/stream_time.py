"""Streaming solver on cfg2 (512 bricks by default): time, G voxel-iter/s, per-kernel ms."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200 import api
import workloads as wl
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = wl.cfg2(batch=B, workers=8)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
out = {}
def run():
    with rwb.solver("streaming"), rwb.stream_passes(passes):
        out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol, max_iter=p.max_iter))
run(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); run(); run(); e.record(); torch.cuda.synchronize()
ms_noprof = s.elapsed_time(e) / 2
api.profile_enable(True)
s.record(); run(); run(); e.record(); torch.cuda.synchronize()
prof = api.profile_read(); api.profile_enable(False)
ms = s.elapsed_time(e) / 2
it = out["iters"].cpu().numpy()
print(json.dumps({"B": B, "passes": passes, "ms_noprof": ms_noprof, "launches": {k: v[0] / 2 for k, v in prof.items() if v[0] > 0}, "ms": ms, "G_voxit_s": float(it.sum()) * 64 ** 3 / ms / 1e6,
                  "kernels": {k: round(v[1] / 2, 2) for k, v in prof.items() if v[1] > 0}}))
