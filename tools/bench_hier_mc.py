#!/usr/bin/env python
"""Multi-class hierarchical random walker (rw_hier_segment_labels).

    python tools/bench_hier_mc.py [--d 1024] [--K 4] [--s 32] [--e 1.25]

Synthetic stand-in for the paper's CT-ORG demonstration (seeds in lungs, liver,
kidneys and background, K = 4): K-1 disjoint "organ" ellipsoids of mean intensity 0.5 .. 0.9 in a
background of 0.15, Gaussian noise sigma 0.04 (the cfg4 recipe) at
u16, generated on the GPU from a fixed seed; 100 seeds per class.  Prints one JSON line per
run: full multi-class run with H_p (homogeneity pruning only), the incremental rerun after
adding 20 seeds of one class, and per-class solved-brick counts.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_09564_b200 as rwb  # noqa: E402


def phantom(d, K, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    rng = np.random.default_rng([31, seed])
    ax = torch.arange(d, device="cuda", dtype=torch.float32) + 0.5
    vol = torch.full((d, d, d), 0.15, device="cuda")
    organs = []
    for k in range(1, K):
        th = 2 * np.pi * k / (K - 1)          # disjoint organs on a ring
        c = (0.5 + np.array([0.1 * (-1) ** k, 0.24 * np.sin(th), 0.24 * np.cos(th)])) * d
        r = rng.uniform(0.08, 0.13, 3) * d
        mu = 0.5 + 0.4 * (k - 1) / max(K - 2, 1)   # organs 0.5 .. 0.9 vs background 0.15
        for z0 in range(0, d, 64):
            z = ax[z0:z0 + 64, None, None]
            q = ((z - c[0]) / r[0]) ** 2 + ((ax[None, :, None] - c[1]) / r[1]) ** 2 + \
                ((ax[None, None, :] - c[2]) / r[2]) ** 2
            vol[z0:z0 + 64][q < 1] = mu
        organs.append((c, r))
    for z0 in range(0, d, 64):
        sl = vol[z0:z0 + 64]
        sl += 0.04 * torch.randn(sl.shape, device="cuda", generator=g)
    vol = (vol.clamp_(0, 1) * 65535).round_().to(torch.int32).to(torch.uint16)
    labels = torch.zeros((d, d, d), dtype=torch.uint8, device="cuda")
    for k, (c, r) in enumerate(organs, start=1):
        u = rng.normal(size=(100, 3))
        u = u / np.linalg.norm(u, axis=1, keepdims=True) * rng.uniform(0, 0.6, (100, 1))
        p = np.clip(np.floor(c + u * r), 0, d - 1).astype(np.int64)
        labels[p[:, 0], p[:, 1], p[:, 2]] = k
    bg = rng.integers(2, d - 2, (400, 3))
    for z, y, x in bg:
        if all(np.sum(((np.array([z, y, x]) + 0.5 - c) / r) ** 2) > 1.2 for c, r in organs):
            labels[z, y, x] = K
    return vol, labels, organs


def timed(fn):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    o = fn()
    t1.record()
    torch.cuda.synchronize()
    return o, t0.elapsed_time(t1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--K", type=int, default=4)
    ap.add_argument("--s", type=int, default=32)
    ap.add_argument("--e", type=float, default=1.25)
    ap.add_argument("--no-state", action="store_true",
                    help="keep neither class fields nor per-class workspaces (no H_it rerun)")
    a = ap.parse_args()
    keep = not a.no_state
    vol, labels, organs = phantom(a.d, a.K)
    kw = dict(s=a.s, e=a.e, tol=1e-6, max_iter=5000)
    o, _ = timed(lambda: rwb.hier_segment_labels(vol, labels, a.K, keep_state=keep,
                                                 keep_prob=keep, **kw))
    ws = o["state"]["workspace"]
    o, ms = timed(lambda: rwb.hier_segment_labels(vol, labels, a.K, keep_state=keep,
                                                  keep_prob=keep, workspace=ws, **kw))
    solved = [sum(st["solved"]) for st in o["stats"]]
    # organ accuracy on voxels well inside / outside each ellipsoid
    lab = o["labels"]
    acc = []
    ax = torch.arange(a.d, device="cuda", dtype=torch.float32) + 0.5
    z = ax[::8, None, None]
    sub = lab[::8, ::8, ::8]
    for k, (c, r) in enumerate(organs, start=1):
        q = ((z - c[0]) / r[0]) ** 2 + ((ax[None, ::8, None] - c[1]) / r[1]) ** 2 + \
            ((ax[None, None, ::8] - c[2]) / r[2]) ** 2
        inside = q < 0.8
        acc.append(float((sub[inside] == k).float().mean()))
    print(json.dumps({"what": "hier_labels", "d": a.d, "K": a.K, "s": a.s, "e": a.e, "ms": round(ms, 2),
                      "out_voxels_per_s": a.d ** 3 / (ms * 1e-3), "solved_per_class": solved,
                      "organ_inside_acc": acc}))
    if not keep:
        return
    new = labels.clone()
    c, r = organs[0]
    rng = np.random.default_rng(99)
    u = rng.normal(size=(20, 3))
    u = u / np.linalg.norm(u, axis=1, keepdims=True) * 0.5
    p = np.clip(np.floor(c + u * r), 0, a.d - 1).astype(np.int64)
    new[p[:, 0], p[:, 1], p[:, 2]] = 1
    o2, ms2 = timed(lambda: rwb.hier_segment_labels(vol, new, a.K, prev=o["state"], **kw))
    print(json.dumps({"what": "hier_labels_incremental", "d": a.d, "K": a.K, "ms": round(ms2, 2),
                      "solved_per_class": [sum(st["solved"]) for st in o2["stats"]],
                      "reused_per_class": [sum(st["reused"]) for st in o2["stats"]]}))


if __name__ == "__main__":
    main()
