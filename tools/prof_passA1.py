"""One cfg3 streaming solve capped at 24 iterations (for ncu of a steady-state k_passA launch).
argv[1]: passes (1 or 2)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
import workloads as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = wl.cfg3()
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rwb.set_device_loop(False)
with rwb.solver("streaming"), rwb.stream_passes(n):
    o = rwb.solve_bricks(d(p.fixed), d(p.values), vol=d(p.vol), beta=p.beta, eps=p.eps, tol=p.tol,
                         max_iter=24, norm=(p.scale, p.offset))
torch.cuda.synchronize()
print("ok", int(o["iters"][0, 0]))
