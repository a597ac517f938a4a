"""Streaming solver: device-driven loop (CUDA graph WHILE node) vs host-driven loop on the
cfg2 batch, cfg3 and cfg4 -- time (CUDA events), bitwise equality, host-side call time."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200 import api
import workloads as wl

d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()


def timed(run, reps=3):
    run(); torch.cuda.synchronize()
    ts, hs = [], []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); t = time.perf_counter(); run(); hs.append((time.perf_counter() - t) * 1e3)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.median(hs))


def solve_case(name, p):
    vol, fixed, values = d(p.vol), d(p.fixed), d(p.values)
    ws = api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, p.dims, p.nrhs), "cuda")
    res = {}
    for mode in (True, False):
        out = {}
        def run():
            out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                        max_iter=p.max_iter, workspace=ws, labels=True,
                                        norm=(p.scale, p.offset)))
        with rwb.solver("streaming"), rwb.device_loop(mode):
            ms, hms = timed(run)
        res[mode] = (ms, hms, {k: v.clone() for k, v in out.items() if v is not None})
    eq = all(torch.equal(res[True][2][k], res[False][2][k]) for k in res[True][2])
    it = res[True][2]["iters"].cpu().numpy()
    print(json.dumps({"case": name, "device_loop_ms": res[True][0], "host_loop_ms": res[False][0],
                      "device_loop_host_call_ms": res[True][1], "host_loop_host_call_ms": res[False][1],
                      "bitwise_equal": bool(eq), "iters_max": int(it.max())}), flush=True)


solve_case("cfg2 512 x 64^3", wl.cfg2(batch=512, workers=16))
solve_case("cfg2 64 x 64^3", wl.cfg2(bricks=list(range(64))))
solve_case("cfg3 512x512x256", wl.cfg3())
lp = wl.cfg4()
seeds, vol = d(lp.labels), d(lp.vol)
ws = api.alloc_workspace(rwb.solve_labels_workspace_bytes(1, lp.dims, lp.K), "cuda")
r = {}
for mode in (True, False):
    out = {}
    def run():
        out.update(rwb.solve_labels(seeds, lp.K, vol=vol, beta=lp.beta, eps=lp.eps, tol=lp.tol,
                                    max_iter=lp.max_iter, workspace=ws))
    with rwb.device_loop(mode):
        ms, hms = timed(run, reps=2)
    r[mode] = (ms, hms, {k: v.clone() for k, v in out.items()})
eq = all(torch.equal(r[True][2][k], r[False][2][k]) for k in r[True][2])
print(json.dumps({"case": "cfg4 256^3 K=4", "device_loop_ms": r[True][0], "host_loop_ms": r[False][0],
                  "device_loop_host_call_ms": r[True][1], "bitwise_equal": bool(eq)}), flush=True)
