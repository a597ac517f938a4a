"""Streaming solver z-chunk sweep on cfg3 / cfg4 (RW_OPT_STREAM_ZC): time, iterations, max |dp|
against the default chunk.   python tools/zc_sweep.py [zc ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb  # noqa: E402
from paper_2103_09564_b200 import api  # noqa: E402
import workloads as wl  # noqa: E402
from tools.bench_configs import ev_time, dev  # noqa: E402

zcs = [int(a) for a in sys.argv[1:]] or [0, 64, 48, 32, 24, 16]


def cfg3():
    p = wl.cfg3()
    vol, fixed, values = dev(p.vol), dev(p.fixed), dev(p.values)
    nx, ny, nz = p.dims
    ref = None
    for zc in zcs:
        with rwb.stream_zc(zc):
            ws = api.alloc_workspace(rwb.solve_workspace_bytes(1, (nx, ny, nz), 1), "cuda")
            out = {}

            def run():
                out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps,
                                            tol=p.tol, max_iter=p.max_iter, workspace=ws))
            ms = ev_time(run, reps=2)
        x = out["prob"].float()
        if ref is None:
            ref = x.clone()
        it = int(out["iters"].max())
        print(json.dumps({"cfg": "cfg3", "zc": zc, "ms": ms, "iters": it,
                          "G": it * nx * ny * nz / ms / 1e6,
                          "maxdp_vs_first": float((x - ref).abs().max())}), flush=True)
        del ws


def cfg4():
    lp = wl.cfg4(n=256)
    seeds, vol = dev(lp.labels), dev(lp.vol)
    ref = None
    for zc in zcs:
        with rwb.stream_zc(zc):
            ws = api.alloc_workspace(rwb.solve_labels_workspace_bytes(1, lp.dims, lp.K), "cuda")
            out = {}

            def run():
                out.update(rwb.solve_labels(seeds, lp.K, vol=vol, beta=lp.beta, eps=lp.eps,
                                            tol=lp.tol, max_iter=lp.max_iter, workspace=ws))
            ms = ev_time(run, reps=2)
        x = out["prob"].float()
        if ref is None:
            ref = x.clone()
        print(json.dumps({"cfg": "cfg4", "zc": zc, "ms": ms,
                          "iters": out["iters"].cpu().numpy().ravel().tolist(),
                          "maxdp_vs_first": float((x - ref).abs().max())}), flush=True)
        del ws


if __name__ == "__main__":
    cfg3()
    cfg4()
