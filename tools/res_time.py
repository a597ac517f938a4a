"""Time the resident vs streaming solver on the cfg2 batch (CUDA events, inputs resident)."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200 import api
import workloads as wl

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = wl.cfg2(batch=nb)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
ws = api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, p.dims, 1), "cuda")
res = {}
for name in ("resident", "streaming"):
    with rwb.solver(name):
        out = {}
        def run():
            out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                        max_iter=p.max_iter, labels=True, workspace=ws))
        run(); torch.cuda.synchronize()
        api.profile_enable(True)
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        prof = api.profile_read(); api.profile_enable(False)
        it = out["iters"].cpu().numpy()
        ms = float(np.median(ts))
        res[name] = dict(ms=ms, iters_sum=int(it.sum()), vox_it_per_s=float(it.sum()) * 64**3 / (ms / 1e3),
                         prob=out["prob"].cpu().numpy(), it=it,
                         kernels={k: v for k, v in prof.items() if v[0] > 0})
        print(json.dumps({"solver": name, "ms": ms, "G_voxit_s": res[name]["vox_it_per_s"] / 1e9,
                          "iters": [int(it.min()), float(np.median(it)), int(it.max())],
                          "kernels": res[name]["kernels"]}), flush=True)
a, b = res["resident"], res["streaming"]
if os.environ.get("RES_DUMP"):     # A/B: keep the resident outputs for a bitwise comparison
    np.savez(os.environ["RES_DUMP"], prob=a["prob"], it=a["it"])
print(json.dumps({"max_abs_dprob": float(np.abs(a["prob"] - b["prob"]).max()),
                  "max_abs_diters": int(np.abs(a["it"].astype(int) - b["it"].astype(int)).max()),
                  "speedup": b["ms"] / a["ms"]}))
