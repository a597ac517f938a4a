"""Small invocations of every device path, for compute-sanitizer (one tool per run)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2103_09564_b200 as rwb
import workloads as wl
from test_hier_oracle import small_volume

d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
p = wl.random_brick(32, 32, 32, seed=1, batch=3, nseed=500, continuous=True, dtype="u16")
for solver in ("streaming", "resident"):
    with rwb.solver(solver):
        o = rwb.solve_bricks(d(p.fixed), d(p.values), vol=d(p.vol), tol=1e-6, labels=True)
q = wl.random_brick(20, 9, 7, seed=2, batch=2, nseed=20, nrhs=3)
rwb.solve_bricks(d(q.fixed), d(q.values), vol=d(q.vol), tol=1e-6)
for kind in ("poisson", "gaussian", "ttest"):
    rwb.brick_weights_ex(d(p.vol), kind=kind)
vol, seeds = small_volume(64, 3)
rwb.hier_segment(d(vol), d(seeds), s=16, e=1.25)
rwb.hier_segment(d(vol), d(seeds), s=16, e=2.0)
rwb.build_pyramid(d(wl.pyramid_volume(40, 36, 34, "u16", seed=0)), 2)
torch.cuda.synchronize()
print("sanitize_small ok")
