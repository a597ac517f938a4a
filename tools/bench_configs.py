#!/usr/bin/env python
"""Per-config measurements beyond bench.py's headline (BASELINE.json configs 1, 3, 4, 5).

    python tools/bench_configs.py [--cfg 1 3 4 5] [--check]

Prints one JSON line per config: solve time (CUDA events, inputs resident), iterations,
voxel-CG-iterations/s, and for the pyramid/queue GB/s.  --check adds property checks at full
size through the oracle (true fp64 residual of the GPU solution for cfg3; sum/argmax sanity
for cfg4) -- slow on the host, off by default.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2103_09564_b200 as rwb  # noqa: E402
from paper_2103_09564_b200 import api  # noqa: E402
import workloads as wl  # noqa: E402


def ev_time(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def solve_cfg(p, name, check=False):
    vol, fixed, values = dev(p.vol), dev(p.fixed), dev(p.values)
    nx, ny, nz = p.dims
    ws = api.alloc_workspace(rwb.solve_workspace_bytes(p.batch, (nx, ny, nz), p.nrhs), "cuda")
    out = {}

    def run():
        out.update(rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                                    max_iter=p.max_iter, labels=True, workspace=ws))
    api.profile_enable(True)
    ms = ev_time(run, reps=3)
    prof = api.profile_read()
    api.profile_enable(False)
    it = out["iters"].cpu().numpy()
    st = out["status"].cpu().numpy()
    vi = float(it.sum()) * nx * ny * nz
    line = {"config": name, "dims": [nx, ny, nz], "batch": p.batch, "ms": ms,
            "iters": {"min": int(it.min()), "max": int(it.max()), "mean": float(it.mean())},
            "status": sorted(set(st.ravel().tolist())),
            "voxel_cg_iter_per_s": vi / (ms / 1e3),
            "kernel_ms_per_solve": {k: v[1] / 4 for k, v in prof.items() if v[1] > 0},
            "launches_per_solve": {k: v[0] // 4 for k, v in prof.items() if v[0] > 0}}
    if check:
        from oracle import rw_oracle as ro
        x = out["prob"].cpu().numpy()[0, 0]
        t = time.time()
        line["true_rel_residual_fp64"] = float(ro.true_residual(p, x))
        line["check_s"] = time.time() - t
        fx = p.fixed[0] > 0
        line["max_principle_ok"] = bool(x.min() >= 0 and x.max() <= 1)
    return line


def cfg4_line(n=256, check=False):
    lp = wl.cfg4(n=n)
    seeds, vol = dev(lp.labels), dev(lp.vol)
    ws = api.alloc_workspace(rwb.solve_labels_workspace_bytes(1, lp.dims, lp.K), "cuda")
    out = {}

    def run():
        out.update(rwb.solve_labels(seeds, lp.K, vol=vol, beta=lp.beta, eps=lp.eps, tol=lp.tol,
                                    max_iter=lp.max_iter, workspace=ws))
    api.profile_enable(True)
    ms = ev_time(run, reps=3)
    prof = api.profile_read()
    api.profile_enable(False)
    it = out["iters"].cpu().numpy()
    vi = float(it.sum()) * n ** 3
    prob = out["prob"].cpu().numpy()
    lab = out["labels"].cpu().numpy()
    line = {"config": f"cfg4 K=4 {n}^3 (3 RHS, shared operator)", "ms": ms,
            "iters_per_rhs": it.ravel().tolist(), "voxel_rhs_cg_iter_per_s": vi / (ms / 1e3),
            "kernel_ms_per_solve": {k: v[1] / 4 for k, v in prof.items() if v[1] > 0},
            "derived_class_min": float(1 - prob.sum(0).max()),
            "seed_labels_kept": bool(np.array_equal(lab[lp.labels > 0], lp.labels[lp.labels > 0]))}
    return line


def pyramid_lines():
    lines = []
    for d in (1024, 2048):
        g = torch.Generator(device="cuda").manual_seed(5)
        vol = torch.randint(0, 65536, (d, d, d), dtype=torch.int32, device="cuda",
                            generator=g).to(torch.uint16)
        levels = 5
        outs = rwb.build_pyramid(vol, levels)
        ms = ev_time(lambda: rwb.build_pyramid(vol, levels, outs=outs), reps=5)
        nbytes = vol.numel() * 2 + sum(o.numel() * 2 for o in outs)
        lines.append({"config": f"pyramid resident {d}^3 u16 -> {levels} levels (fused)",
                      "ms": ms, "GBps": nbytes / (ms / 1e3) / 1e9,
                      "alg_bytes": nbytes})
        del vol, outs
        torch.cuda.empty_cache()
    # streamed through the pinned double-buffered queue (cfg5 shape at 1/2 scale)
    d = 1024
    slab = 32
    levels = 5
    host = np.random.default_rng(5).integers(0, 65536, (d, d, d), dtype=np.uint16)
    outs = [torch.empty((z, y, x), dtype=torch.uint16, device="cuda")
            for (x, y, z) in api.level_dims((d, d, d), levels)]
    q = rwb.Queue(slab * d * d * 2, depth=3)
    cs = torch.cuda.Stream()
    ms_stream = torch.cuda.current_stream()

    def stream_all():
        for z0 in range(0, d, slab):
            ptr, sid = q.push(host[z0:z0 + slab], cs)
            q.wait(sid, ms_stream)
            t = api.device_view(ptr, (slab, d, d), torch.uint16, "cuda")
            rwb.build_pyramid_slab(t, (d, d, d), z0, levels, outs)
            q.release(sid, ms_stream)
    stream_all()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stream_all()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ref = rwb.build_pyramid(torch.from_numpy(host).cuda(), levels)
    same = all(torch.equal(a, b) for a, b in zip(outs, ref))
    lines.append({"config": f"pyramid streamed {d}^3 u16 via rw_queue (32-plane slabs, depth 3)",
                  "wall_ms": wall * 1e3, "host_GBps": host.nbytes / wall / 1e9,
                  "equals_resident": bool(same)})
    q.close()
    return lines


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", nargs="*", type=int, default=[1, 3, 4, 5])
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    if 1 in a.cfg:
        print(json.dumps(solve_cfg(wl.cfg1(), "cfg1 32^3 f32 sphere", a.check)), flush=True)
        rwb.set_resident_wide(True)       # latency-shaped 8-CTA cluster for the single brick
        try:
            print(json.dumps(solve_cfg(wl.cfg1(), "cfg1 32^3 f32 sphere (RW_OPT_RESIDENT_WIDE)",
                                       a.check)), flush=True)
        finally:
            rwb.set_resident_wide(False)
    if 3 in a.cfg:
        p = wl.cfg3()
        print(json.dumps(solve_cfg(p, "cfg3 512x512x256 i16 CT phantom", a.check)), flush=True)
    if 4 in a.cfg:
        print(json.dumps(cfg4_line(256, a.check)), flush=True)
    if 5 in a.cfg:
        for ln in pyramid_lines():
            print(json.dumps(ln), flush=True)


if __name__ == "__main__":
    main()
