"""Streaming CG with one vs two HBM passes per iteration (RW_OPT_STREAM_PASSES) on cfg2
(64 bricks), cfg3 and cfg4: time (CUDA events), iterations, per-kernel ms, max |dp|."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
from paper_2103_09564_b200 import api
import workloads as wl


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def timed(fn, reps):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    api.profile_enable(True)
    s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    prof = api.profile_read(); api.profile_enable(False)
    return s.elapsed_time(e) / reps, {k: round(v[1] / reps, 3) for k, v in prof.items() if v[1] > 0}


def case(name, run, reps):
    res = {}
    for n in (2, 1):
        with rwb.solver("streaming"), rwb.stream_passes(n):
            ms, prof = timed(run, reps)
            o = run(); torch.cuda.synchronize()
        res[n] = (ms, prof, o["prob"].cpu().numpy(), o["iters"].cpu().numpy())
    d = float(np.abs(res[1][2] - res[2][2]).max())
    di = int(np.abs(res[1][3].astype(int) - res[2][3].astype(int)).max())
    print(json.dumps({"case": name, "ms_2pass": res[2][0], "ms_1pass": res[1][0],
                      "speedup": res[2][0] / res[1][0], "kernels_2pass": res[2][1],
                      "kernels_1pass": res[1][1], "iters_2pass": [int(res[2][3].min()), int(res[2][3].max())],
                      "iters_1pass": [int(res[1][3].min()), int(res[1][3].max())],
                      "max_abs_dprob": d, "max_abs_diters": di}), flush=True)


p = wl.cfg2(batch=64)
vol, fixed, values = dev(p.vol), dev(p.fixed), dev(p.values)
case("cfg2 64 bricks", lambda: rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                                max_iter=p.max_iter), 3)
p3 = wl.cfg3()
v3, f3, x3 = dev(p3.vol), dev(p3.fixed), dev(p3.values)
case("cfg3", lambda: rwb.solve_bricks(f3, x3, vol=v3, beta=p3.beta, eps=p3.eps, tol=p3.tol,
                                      max_iter=p3.max_iter, norm=(p3.scale, p3.offset)), 1)
lp = wl.cfg4()
l4, v4 = dev(lp.labels), dev(lp.vol)
case("cfg4", lambda: rwb.solve_labels(l4, lp.K, vol=v4, beta=lp.beta, eps=lp.eps, tol=lp.tol,
                                      max_iter=lp.max_iter), 1)
