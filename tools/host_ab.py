"""rw_solve_bricks_host on cfg2: the streamed resident path (one persistent launch, chunk
flags) vs the chunked path (RW_HOST_CHUNKED=1), bitwise against the device solve, e2e time.
    python tools/host_ab.py [B] [chunk ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb  # noqa: E402
from paper_2103_09564_b200 import api  # noqa: E402
import workloads as wl  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
chunks = [int(a) for a in sys.argv[2:]] or [0]
p = wl.cfg2(batch=B, workers=16)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ref = rwb.solve_bricks(d(p.fixed), d(p.values), vol=d(p.vol), beta=p.beta, eps=p.eps, tol=p.tol,
                       max_iter=p.max_iter, labels=True)
torch.cuda.synchronize()
ref = {k: v.cpu() for k, v in ref.items() if v is not None}
vi = float(ref["iters"].sum()) * 64 ** 3
hv, hf, hx = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (p.vol, p.fixed, p.values[0]))
out = dict(prob=torch.empty((1,) + tuple(hf.shape), dtype=torch.float32).pin_memory(),
           labels=torch.empty(tuple(hf.shape), dtype=torch.uint8).pin_memory(),
           iters=torch.empty((1, B), dtype=torch.int32).pin_memory(),
           resid=torch.empty((1, B), dtype=torch.float32).pin_memory(),
           status=torch.empty((1, B), dtype=torch.int32).pin_memory())
for mode in ("streamed", "chunked"):
    if mode == "chunked":
        os.environ["RW_HOST_CHUNKED"] = "1"
    for ch in chunks:
        ws = api.alloc_workspace(api.lib().rw_solve_host_workspace_bytes(
            B, api.rw_dims(64, 64, 64), api.DTYPES[torch.uint16], ch), "cuda")
        run = lambda: rwb.solve_bricks_host(hf, hx, hv, beta=p.beta, eps=p.eps, tol=p.tol,
                                            max_iter=p.max_iter, chunk=ch, prob=True, labels=True,
                                            workspace=ws, out=out)
        run()
        torch.cuda.synchronize()
        eq = {k: bool(torch.equal(out[k], ref[k])) for k in ("prob", "labels", "iters", "resid", "status")}
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        ms = float(np.median(ts))
        print(json.dumps({"mode": mode, "B": B, "chunk": ch, "ms": ms, "G": vi / ms / 1e6,
                          "ms_all": ts, "bitwise_equal_device": eq}), flush=True)
        del ws
    os.environ.pop("RW_HOST_CHUNKED", None)
