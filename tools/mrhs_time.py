"""Multi-label bricks (K = 4 -> 3 rhs on one operator): resident (rhs, brick) pairs vs the
streaming shared-operator passes.  B copies of the cfg4 recipe at n^3.
    python tools/mrhs_time.py [n] [B]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb  # noqa: E402
from paper_2103_09564_b200 import api  # noqa: E402
import workloads as wl  # noqa: E402
from tools.bench_configs import ev_time  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
lp = wl.cfg4(n=n, seeds_per_label=max(20, n // 2))
seeds = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(lp.labels, (B,) + lp.labels.shape[-3:]))).cuda()
vol = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(lp.vol, (B,) + lp.vol.shape[-3:]))).cuda()
ws = api.alloc_workspace(rwb.solve_labels_workspace_bytes(B, (n, n, n), lp.K), "cuda")
res = {}
for name in ("resident", "streaming"):
    out = {}

    def run():
        with rwb.solver(name):
            out.update(rwb.solve_labels(seeds, lp.K, vol=vol, beta=lp.beta, eps=lp.eps, tol=lp.tol,
                                        max_iter=lp.max_iter, workspace=ws))
    ms = ev_time(run, reps=3)
    it = out["iters"].cpu().numpy()
    res[name] = (ms, out["prob"].clone())
    print(json.dumps({"solver": name, "n": n, "B": B, "rhs": lp.K - 1, "ms": ms,
                      "iters_rhs": it[:, 0].tolist(),
                      "G_voxel_rhs_iter_per_s": float(it.sum()) * n ** 3 / ms / 1e6}), flush=True)
print(json.dumps({"max_dp_resident_vs_streaming": float((res["resident"][1] - res["streaming"][1]).abs().max())}))
