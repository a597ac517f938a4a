#!/usr/bin/env python
"""Hierarchical random walker (rw_hier_segment) on the config-5 vessel volume.

    python tools/bench_hier.py [--scale 0.25] [--s 32] [--e 1.25] [--no-prune-too]

Generates the seeded synthetic vessel network of BASELINE.json config 5 at `scale` (2048^3 x
scale), rasterised seeds (foreground on vessel centre lines, background in vessel-free
spots), runs H_p (pruning on) and optionally plain H (no pruning), and prints one JSON line
per run: wall time (CUDA events, inputs resident), per-level brick statistics, output
voxels/s and solved-brick voxel-CG-iterations.
"""
import argparse
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_09564_b200 as rwb  # noqa: E402
import workloads as wl  # noqa: E402
from workloads.gen import _vessel_segments  # noqa: E402


def volume(scale, workers=16):
    return wl.cfg5_volume(scale, workers)


def seed_labels(vol, scale, nfg=400, nbg=400, seed=0):
    return wl.cfg5_seeds(vol, nfg, nbg, seed)


def run(vol_d, seeds_d, s, e, prune, reps=2, prev=None, ws=None, prob_buf=None):
    out = None
    ts = []
    for _ in range(reps + 1):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        prob, st, state = rwb.hier_segment(vol_d, seeds_d, s=s, e=e, prune=prune, tol=1e-6,
                                           max_batch=int(os.environ.get("HIER_MAX_BATCH", "1024")),
                                           max_iter=5000, workspace=ws, prev=prev, out=prob_buf)
        t1.record()
        torch.cuda.synchronize()
        ts.append(t0.elapsed_time(t1))
        ws = state["workspace"]
        prob_buf = prob
        out = (prob, st, state)
        if prev is not None:
            break          # an incremental update is measured once (it changes the state)
    return out, float(np.median(ts[1:] if len(ts) > 1 else ts))


def new_seeds(vol, seeds, n=50, seed=1):
    return wl.cfg5_new_seeds(vol, seeds, n, seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.25)
    ap.add_argument("--s", type=int, default=32)
    ap.add_argument("--e", type=float, default=1.25)
    ap.add_argument("--no-prune-too", action="store_true")
    a = ap.parse_args()
    t = time.time()
    vol = volume(a.scale)
    seeds = seed_labels(vol, a.scale)
    d = vol.shape[0]
    print(f"[bench_hier] generated {d}^3 in {time.time() - t:.1f}s; seeds fg {(seeds == 1).sum()} "
          f"bg {(seeds == 2).sum()}", file=sys.stderr, flush=True)
    vol_d = torch.from_numpy(vol).cuda()
    seeds_d = torch.from_numpy(seeds).cuda()
    se = int(math.floor(a.e * a.s))
    runs = [True] + ([False] if a.no_prune_too else [])
    res = {}
    ws = buf = None
    from paper_2103_09564_b200 import api
    for prune in runs:
        api.profile_enable(True)
        (prob, st, state), ms = run(vol_d, seeds_d, a.s, a.e, prune, ws=ws, prob_buf=buf)
        prof = api.profile_read()
        api.profile_enable(False)
        ws, buf = state["workspace"], prob
        total = sum((d // a.s >> l) ** 3 for l in range(st["levels"]))
        vi = sum(st["iters"][l] * se ** 3 for l in range(st["levels"] - 1)) + st["iters"][-1] * a.s ** 3
        line = {"config": f"cfg5 vessels {d}^3 u16, hierarchical (s={a.s}, e={a.e}, s_e={se})",
                "prune": prune, "ms": ms, "output_voxels_per_s": d ** 3 / (ms / 1e3),
                "bricks_solved": sum(st["solved"]), "bricks_total": total,
                "solved_voxel_cg_iter_per_s": vi / (ms / 1e3), "stats": st,
                "fg_fraction": float((prob > 0.5).float().mean()),
                "kernel_ms_all_reps": {k: round(v[1], 2) for k, v in prof.items() if v[1] > 0},
                "launches_all_reps": {k: v[0] for k, v in prof.items() if v[0] > 0}}
        if a.no_prune_too:
            res[prune] = (prob > 0.5).cpu() if d > 1024 else prob.clone()
        print(json.dumps(line), flush=True)
        if prune:
            # config 5's incremental update: 50 new seeds (H_it)
            seeds2 = new_seeds(vol, seeds)
            (prob2, st2, _), ms2 = run(vol_d, torch.from_numpy(seeds2).cuda(), a.s, a.e, True,
                                       prev=state)
            if a.no_prune_too:   # the unpruned run below starts from scratch on the same buffers
                pass
            print(json.dumps({"config": line["config"] + " incremental +50 fg seeds",
                              "ms": ms2, "bricks_solved": sum(st2["solved"]),
                              "bricks_reused": sum(st2["reused"]), "stats": st2}), flush=True)
    if len(res) == 2:
        A, B = res[True], res[False]
        if A.dtype == torch.bool:
            print(json.dumps({"label_agreement": float((A == B).float().mean())}), flush=True)
        else:
            print(json.dumps({"pruned_vs_full_max_abs": float((A - B).abs().max()),
                              "label_agreement": float(((A > 0.5) == (B > 0.5)).float().mean())}), flush=True)


if __name__ == "__main__":
    main()
