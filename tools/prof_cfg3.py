"""One cfg3 (512x512x256 i16) streaming solve capped at 24 iterations, host-driven loop
(for ncu of a steady-state k_passA launch)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
import workloads as wl
p = wl.cfg3()
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rwb.set_device_loop(False)
o = rwb.solve_bricks(d(p.fixed), d(p.values), vol=d(p.vol), beta=p.beta, eps=p.eps, tol=p.tol,
                     max_iter=24)
torch.cuda.synchronize()
print("ok", o["iters"].cpu().numpy().ravel().tolist())
