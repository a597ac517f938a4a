import os, sys, json
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200 import api
from paper_2103_09564_b200._lib import lib
import workloads as wl
p = wl.cfg2(batch=64)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
ws = api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, p.dims, 1), "cuda")
res = {}
for pm in (0, 250):
    lib().rw_set_option(1, pm)
    o = rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol, max_iter=p.max_iter, workspace=ws)
    torch.cuda.synchronize()
    res[pm] = {k: (v.cpu().numpy() if v is not None else None) for k, v in o.items()}
a, b = res[0], res[250]
dp = np.abs(a["prob"] - b["prob"]).reshape(64, -1).max(1)
print("per-brick max dp:", np.round(dp, 6).tolist())
print("iters0", a["iters"].ravel().tolist())
print("iters1", b["iters"].ravel().tolist())
print("status1", b["status"].ravel().tolist())
with rwb.solver("streaming"):
    lib().rw_set_option(1, 0)
    o = rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol, max_iter=p.max_iter, workspace=ws)
    torch.cuda.synchronize()
print("streaming-only vs pm250 tail:", np.abs(o["prob"].cpu().numpy() - b["prob"]).reshape(64,-1).max(1)[-20:].round(6).tolist())
