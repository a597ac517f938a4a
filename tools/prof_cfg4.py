"""One cfg4 (256^3, K = 4) streaming multi-rhs solve capped at 24 iterations, host-driven loop
(for ncu of a steady-state k_passA launch)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
import workloads as wl
lp = wl.cfg4(n=256)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rwb.set_device_loop(False)
o = rwb.solve_labels(d(lp.labels), lp.K, vol=d(lp.vol), beta=lp.beta, eps=lp.eps, tol=lp.tol, max_iter=24)
torch.cuda.synchronize()
print("ok", o["iters"].cpu().numpy().ravel().tolist())
