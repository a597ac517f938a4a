#!/usr/bin/env python
"""Out-of-core hierarchical random walker (rw_hier_segment_ooc) on the config-5 vessel network
at sizes beyond what the in-HBM driver can hold.

    python tools/bench_ooc.py --d 4096 --nz 2048 [--compare-hbm] [--prob]

Volume: the config-5 generator (workloads.cfg5_slab, scale d/2048) restricted to planes
[0, nz) -- a d x d x nz u16 volume in host memory (4096 x 4096 x 2048 = 64 GiB); seeds: fg at
vessel-segment mid points inside the volume, bg at vessel-free random voxels.  Prints one JSON
line: volume, phase wall times, per-level solve / prune counts, brick-pool use, device workspace.
--compare-hbm (cubic volumes that fit): the in-HBM driver on the same volume, labels compared.
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads.gen as gen  # noqa: E402


def volume(d, nz, workers=16):
    scale = d / 2048
    vol = np.empty((nz, d, d), np.uint16)
    gen.cfg5_slab(0, 1, scale)                      # segment cache
    step = max(1, nz // (workers * 8))

    def fill(z):
        vol[z:min(z + step, nz)] = gen.cfg5_slab(z, min(z + step, nz), scale)
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(fill, range(0, nz, step)))
    return vol


def seeds_for(vol, d, nfg=400, nbg=400, seed=0):
    nz = vol.shape[0]
    rng = np.random.default_rng([5, 2, seed])
    seeds = np.zeros(vol.shape, np.uint8)
    segs = gen._vessel_segments(d)
    mids = [np.floor((p0 + p1) / 2).astype(int) for p0, p1, r in segs]
    mids = [m for m in mids if 0 <= m[2] < nz]
    pick = rng.choice(len(mids), size=min(nfg, len(mids)), replace=False)
    for i in pick:
        x, y, z = np.clip(mids[i], 0, [d - 1, d - 1, nz - 1])
        if vol[z, y, x] > 15000:
            seeds[z, y, x] = 1
    n = 0
    while n < nbg:
        z = rng.integers(2, nz - 2)
        y, x = rng.integers(2, d - 2, 2)
        if vol[z - 2:z + 3, y - 2:y + 3, x - 2:x + 3].max() < 10000:
            seeds[z, y, x] = 2
            n += 1
    return seeds


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--nz", type=int, default=2048)
    ap.add_argument("--s", type=int, default=32)
    ap.add_argument("--prob", action="store_true", help="also return the fp32 field")
    ap.add_argument("--compare-hbm", action="store_true")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--pinned", action="store_true",
                    help="page-locked volume / seeds / outputs (no host staging copies) and a "
                         "queue + workspace allocated once, outside the timed call")
    ap.add_argument("--no-pin-seeds", action="store_true",
                    help="with --pinned: leave the seed volume pageable (it is only scanned on "
                         "the host; its non-zero segments are staged)")
    a = ap.parse_args()
    import torch
    import paper_2103_09564_b200 as rwb
    t = time.time()
    vol = volume(a.d, a.nz)
    seeds = seeds_for(vol, a.d)
    gen_s = time.time() - t
    kw = dict(s=a.s, e=1.25, t_hom=0.3, t_bin=0.01, prune=True, beta=100.0, tol=1e-6)
    out = None
    walls = []
    pin_s = None
    if a.pinned:
        t = time.time()
        regs = [rwb.host_register(vol)] + ([] if a.no_pin_seeds else [rwb.host_register(seeds)])
        kw["out_labels"] = rwb.pinned_empty(vol.shape, np.uint8)
        if a.prob:
            kw["out_prob"] = rwb.pinned_empty(vol.shape, np.float32)
        kw["queue"], kw["workspace"], kw["pool_bricks"] = rwb.hier_ooc_alloc(vol.shape, vol.dtype, s=a.s)
        pin_s = time.time() - t
    for r in range(a.reps):
        torch.cuda.synchronize()
        t = time.time()
        prob, lab, st = rwb.hier_segment_ooc(vol, seeds, want_prob=a.prob, **kw)
        walls.append(time.time() - t)
        out = (prob, lab, st)
    if a.pinned:
        for r in regs:
            r.close()
        for k in ("out_labels", "out_prob", "queue", "workspace", "pool_bricks"):
            kw.pop(k, None)
    prob, lab, st = out
    line = {"config": f"cfg5 vessel network {a.d}x{a.d}x{a.nz} u16 "
                      f"({vol.nbytes / 2**30:.0f} GiB host), s = {a.s}, e = 1.25, H_p, out of core",
            "generate_s": gen_s, "wall_s": walls, "ms_phases": st["ms"],
            "levels": st["levels"], "solved": st["solved"], "active": st["active"],
            "pruned_hom": st["pruned_hom"], "pruned_dt": st["pruned_dt"],
            "bricks_solved": int(sum(st["solved"])), "pool_used": st["pool_used"],
            "iters": st["iters"], "fg_voxels": int(lab.sum(dtype=np.int64)),
            "output": "fp32 prob + u8 labels" if a.prob else "u8 labels"}
    if a.pinned:
        line["host_buffers"] = ("page-locked (registered volume" + ("" if a.no_pin_seeds else " / seeds") +
                                ", pinned outputs); queue and workspace reused")
        line["pin_and_alloc_s"] = pin_s
    try:
        free, total = torch.cuda.mem_get_info()
        line["device_peak_alloc_GB"] = torch.cuda.max_memory_allocated() / 1e9
    except Exception:
        pass
    if a.compare_hbm and a.d == a.nz:
        v = torch.from_numpy(vol).cuda()
        sd = torch.from_numpy(seeds).cuda()
        del vol
        ref, st2, _ = rwb.hier_segment(v, sd, **kw)
        torch.cuda.synchronize()
        t = time.time()
        ref, st2, _ = rwb.hier_segment(v, sd, **kw)
        torch.cuda.synchronize()
        line["hbm_driver_s"] = time.time() - t
        line["hbm_solved"] = st2["solved"]
        lab2 = (ref > 0.5).to(torch.uint8).cpu().numpy()
        line["labels_equal_hbm_driver"] = bool(np.array_equal(lab2, lab))
        if prob is not None:
            line["prob_equal_hbm_driver"] = bool(np.array_equal(ref.cpu().numpy(), prob))
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
