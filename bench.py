#!/usr/bin/env python
"""Benchmark of the B200 random walker hot path (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]

One step = one ``rw_solve_bricks`` call on the whole config-2 batch (512 independent
64^3 u16 bricks): weights from intensities (a1/a2), implicit assembly (a3), the
Jacobi-PCG loop until every brick has converged (a4/a5), finalise + labels (a6).  Inputs
are resident in HBM (7.5 GB of CG state + inputs, far larger than L2, so no L2 flush is
needed between steps).  value = voxel-CG-iterations/s over all ranks
(sum_b n_b * iters_b / step time), weak scaling (each rank solves its own 512 bricks).

--solver auto (default) lets the library pick: the brick-resident solver (one 16-CTA
cluster per 64^3 brick, CG state on chip) for this shape; --solver streaming forces the
HBM-streaming passes.  When the resident solver is the headline, the streaming solver is
also timed on the same inputs and reported under "streaming" with its HBM roofline.

--impl reference times the fp64 oracle (oracle/, numpy+scipy) on the host cores on a
bounded sample of the same workload -- this tier's reference arm (no reference code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxel-CG-iterations/s"
UNIT = "voxel-CG-iter/s"
WORKLOAD = "cfg2: 512 x 64^3 u16 bricks, 1-5 blobs, Dirichlet shell, 0.1% seeds, beta=100, tol=1e-6 rel, max_iter=2000"
BATCH, N = 512, 64
# algorithmic bytes per active voxel per launch.  Pass A (weights recomputed
# from the u16 intensities, VM_U16) reads r, p, dinv, x (16 B) + the intensity (2 B) and
# writes p, x, q (12 B); at k = 0 there is no x traffic.  Pass B reads r, q, dinv, writes r.
BYTES_A, BYTES_A0, BYTES_B = 30, 22, 16       # two-pass streaming CG (RW_OPT_STREAM_PASSES 2)
BYTES_1, BYTES_10 = 38, 26                      # one-pass (default): pass k >= 1, pass 0
# fp32 flops per voxel-iteration of the resident kernel: edge-difference
# SpMV 6 sub + 6 mul/fma (18), p = dinv r + beta p (3), x += alpha p (2), r -= alpha q (2),
# dots p.q (2), r.(dinv r) (3), r.r (2)
FLOPS_RES = 32
FP32_LANES_PER_SM, SMS = 128, 148


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def make_inputs(rank, world, workers):
    import workloads as wl
    from paper_2103_09564_b200.dist import shard_bricks
    ids = shard_bricks(rank, world, BATCH)
    t = time.time()
    p = wl.cfg2(bricks=ids, n=N, workers=workers)
    log(f"[rank {rank}] generated {len(ids)} bricks in {time.time() - t:.1f}s")
    return p


def cpu_oracle_sample(nbricks, seed0=0):
    """Time the fp64 oracle (as it stands) on ``nbricks`` bricks of the same workload at the
    same tolerance; returns (voxel-iter/s, seconds, voxel-iterations, threads used)."""
    import workloads as wl
    from oracle import rw_oracle as ro
    from threadpoolctl import threadpool_limits
    p = wl.cfg2(bricks=list(range(seed0, seed0 + nbricks)), n=N)
    with threadpool_limits(1):
        t = time.perf_counter()
        o = ro.solve_problem(p, tol=p.tol, max_iter=p.max_iter)
        dt = time.perf_counter() - t
    vi = float(np.sum(o["iters"])) * N ** 3
    return vi / dt, dt, vi, 1


def run_reference(args, rank, world):
    if rank != 0:
        return
    nb = 3
    vals, tot_t = [], 0.0
    for s in range(args.warmup + args.steps):
        v, dt, vi, cores = cpu_oracle_sample(nb, seed0=(s * nb) % BATCH)
        if s >= args.warmup:
            vals.append(v)
            tot_t += dt
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * tot_t / max(1, args.steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": f"{nb} bricks of 64^3 per step (of 512)",
                   "parallelism": "single host thread"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{nb} cfg2 bricks per step, fp64 CSR Jacobi-PCG to rel 1e-6"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def streaming_roofline(kms, vox_iters, steps, nbr):
    """HBM roofline of the streaming passes from the profile of `steps` solves."""
    vox = float(N ** 3)
    one = kms.get("passB", 0.0) == 0.0
    if one:   # one pass per iteration: iters_b full passes + pass 0 per brick (rw.h)
        alg = {"passA": steps * (BYTES_1 * vox_iters + BYTES_10 * vox * nbr), "passB": 0.0}
    else:
        alg = {"passA": steps * (BYTES_A * vox_iters - (BYTES_A - BYTES_A0) * vox * nbr),
               "passB": steps * BYTES_B * vox_iters}
    dom = max(("passA", "passB"), key=lambda k: kms.get(k, 0.0))
    peak, peak_kind = measured_peak()
    achieved = alg[dom] / (kms[dom] / 1000.0) / 1e9
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(dom),
            "per_kernel_ms_per_step": {k: v / steps for k, v in kms.items() if v > 0},
            "alg_bytes_per_voxel_iter": ({"passA": BYTES_1, "passA_k0": BYTES_10} if one else
                                         {"passA": BYTES_A, "passB": BYTES_B}),
            "passes_per_iteration": 1 if one else 2}


def ncu_traffic(kernel):
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(tr_path) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def fp32_peak_tflops():
    """fp32 FMA peak from the unit counts and the measured max SM clock."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz, kind = float(json.load(f)["sm_max_mhz"]), "derived: 148 SMs x 128 fp32 lanes x 2 x measured sm_max_mhz"
    except Exception:
        mhz, kind = 1965.0, "derived: 148 SMs x 128 fp32 lanes x 2 x 1965 MHz (guide)"
    return SMS * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12, kind


def pyramid_and_queue(dev, d=1024, levels=5, slab=128):
    """SURVEY 8(a) rows a8 (LOD pyramid) and a9 (pinned double-buffered queue), measured in
    the same run on a seeded 1024^3 u16 volume: resident fused 5-level pyramid (algorithmic
    bytes = input + all levels) and the volume streamed from pinned host memory in 32-plane
    slabs through rw_queue into rw_build_pyramid_slab (bound: host-to-device copy)."""
    import torch
    import paper_2103_09564_b200 as rwb
    from paper_2103_09564_b200 import api
    g = torch.Generator(device=dev).manual_seed(5)
    vol = torch.randint(0, 65536, (d, d, d), dtype=torch.int32, device=dev, generator=g).to(torch.uint16)
    outs = rwb.build_pyramid(vol, levels)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        rwb.build_pyramid(vol, levels, outs=outs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    nbytes = vol.numel() * 2 + sum(o.numel() * 2 for o in outs)
    peak, kind = measured_peak()
    host = vol.cpu().pin_memory().numpy()     # pinned host volume: no staging copy (rw_queue_push)
    del vol
    q = rwb.Queue(slab * d * d * 2, depth=3)
    cs = torch.cuda.Stream(dev)
    ms_stream = torch.cuda.current_stream(dev)
    outs2 = [torch.empty_like(o) for o in outs]

    def stream_all():
        for z0 in range(0, d, slab):
            ptr, sid = q.push(host[z0:z0 + slab], cs)
            q.wait(sid, ms_stream)
            t = api.device_view(ptr, (slab, d, d), torch.uint16, dev)
            rwb.build_pyramid_slab(t, (d, d, d), z0, levels, outs2)
            q.release(sid, ms_stream)
    stream_all()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stream_all()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    same = all(torch.equal(a, b) for a, b in zip(outs, outs2))
    q.close()
    # roofline of the queue: plain pinned host -> device copy bandwidth of this box
    # (1 GiB copies: smaller pinned copies reach less, e.g. 31 GB/s at 64 MiB, 52 at 256 MiB)
    hp = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    dd = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    dd.copy_(hp, non_blocking=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        dd.copy_(hp, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d_peak = 4 * hp.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
    del hp, dd
    return {"pyramid": {"workload": f"{d}^3 u16 -> {levels} levels (fused, resident)", "ms": ms,
                        "achieved_GBps": nbytes / ms / 1e6, "peak_GBps": peak, "peak_kind": kind,
                        "frac": nbytes / ms / 1e6 / peak},
            "queue": {"workload": f"{d}^3 u16 streamed from pinned host memory, {slab}-plane slabs, "
                                  "depth 3, pyramid per slab", "wall_ms": wall * 1e3,
                      "host_GBps": host.nbytes / wall / 1e9, "equals_resident": bool(same),
                      "bound": "pcie", "peak_GBps": h2d_peak, "peak_kind": "measured pinned H2D copy",
                      "frac": host.nbytes / wall / 1e9 / h2d_peak}}


def run_b200(args, rank, world, local_rank):
    import torch
    import paper_2103_09564_b200 as rwb
    from paper_2103_09564_b200 import api
    from paper_2103_09564_b200.dist import reduce_metric

    dist = None
    if world > 1:
        import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p = make_inputs(rank, world, args.workers)
    vol = torch.from_numpy(p.vol).to(dev)
    fixed = torch.from_numpy(p.fixed).to(dev)
    values = torch.from_numpy(p.values).to(dev)
    need = rwb.solve_workspace_bytes(BATCH, (N, N, N), 1)
    ws = api.alloc_workspace(need, dev)
    out = dict(prob=torch.empty_like(values),
               iters=torch.empty((1, BATCH), dtype=torch.int32, device=dev),
               resid=torch.empty((1, BATCH), dtype=torch.float32, device=dev),
               status=torch.empty((1, BATCH), dtype=torch.int32, device=dev),
               labels=torch.empty(tuple(fixed.shape), dtype=torch.uint8, device=dev))
    stream = torch.cuda.current_stream(dev)

    rwb.set_solver(args.solver)

    def step():
        rwb.solve_bricks(fixed, values, vol=vol, beta=p.beta, eps=p.eps, tol=p.tol,
                         max_iter=p.max_iter, workspace=ws, out=out, stream=stream)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    iters = out["iters"].cpu().numpy().astype(np.int64)
    assert (out["status"].cpu().numpy() == 1).all(), "not all bricks converged"
    vox_iters = float(iters.sum()) * N ** 3

    # ---------------- device-timed region (inputs resident) ----------------
    clk = Clocks(local_rank)
    api.profile_enable(True)
    barrier()
    torch.cuda.synchronize()
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    barrier()
    ms = e0.elapsed_time(e1)
    prof = api.profile_read()
    api.profile_enable(False)
    # max device time over ranks, total work over ranks (paper_2103_09564_b200.dist)
    t_max, work_all = reduce_metric(ms, vox_iters, dev)
    ms_per_step = t_max / args.steps
    value = work_all / (ms_per_step / 1000.0)

    # ---------------- roofline of the dominant kernel ----------------
    launches = {k: v[0] for k, v in prof.items()}
    kms = {k: v[1] for k, v in prof.items()}
    solver_used = "resident" if kms.get("resident", 0.0) > 0 else "streaming"
    if solver_used == "resident":
        peak, peak_kind = fp32_peak_tflops()
        achieved = FLOPS_RES * vox_iters * args.steps / (kms["resident"] / 1000.0) / 1e12
        roofline = {"bound": "alu", "kernel": "resident", "achieved": achieved, "peak": peak,
                    "peak_kind": peak_kind, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": ncu_traffic("resident"),
                    "per_kernel_ms_per_step": {k: v / args.steps for k, v in kms.items() if v > 0},
                    "alg_flops_per_voxel_iter": FLOPS_RES,
                    "note": "CG state on chip for all iterations (no per-iteration HBM traffic); "
                            "bound by on-chip latency: two cluster-wide reductions and a DSMEM "
                            "halo exchange per iteration (DESIGN.md 5)"}
    else:
        roofline = streaming_roofline(kms, vox_iters, args.steps, BATCH)

    streaming = None
    if solver_used == "resident" and not args.no_streaming:
        # the HBM-streaming solver on the same inputs (secondary line: % of HBM peak)
        with rwb.solver("streaming"):
            step()
            torch.cuda.synchronize()
            api.profile_enable(True)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            sms_ = e0.elapsed_time(e1)
            sprof = api.profile_read()
            api.profile_enable(False)
        s_iters = out["iters"].cpu().numpy().astype(np.int64)
        s_vi = float(s_iters.sum()) * N ** 3
        st_max, s_work = reduce_metric(sms_, s_vi, dev)
        streaming = {"value": s_work / (st_max / args.steps / 1000.0), "unit": UNIT,
                     "ms_per_step": st_max / args.steps,
                     "roofline": streaming_roofline({k: v[1] for k, v in sprof.items()}, s_vi,
                                                    args.steps, BATCH),
                     "gpu_launches": int(sum(v[0] for v in sprof.values()))}

    # ---------------- end to end through the API with host buffers ----------------
    # rw_solve_bricks_host: pinned host inputs -> chunked H2D / solve / D2H pipeline -> host
    # labels + iterations (the copies are inside the timed region, overlapped with the solve)
    h_vol = torch.from_numpy(p.vol).pin_memory()
    h_fixed = torch.from_numpy(p.fixed).pin_memory()
    h_values = torch.from_numpy(p.values[0]).pin_memory()
    h_out = dict(prob=None, labels=torch.empty(tuple(fixed.shape), dtype=torch.uint8).pin_memory(),
                 iters=torch.empty((1, BATCH), dtype=torch.int32).pin_memory(),
                 resid=torch.empty((1, BATCH), dtype=torch.float32).pin_memory(),
                 status=torch.empty((1, BATCH), dtype=torch.int32).pin_memory())
    h_ws = api.alloc_workspace(api.lib().rw_solve_host_workspace_bytes(
        BATCH, api.rw_dims(N, N, N), api.DTYPES[torch.uint16], args.e2e_chunk), dev)

    def e2e_step():
        rwb.solve_bricks_host(h_fixed, h_values, h_vol, beta=p.beta, eps=p.eps, tol=p.tol,
                              max_iter=p.max_iter, chunk=args.e2e_chunk, labels=True,
                              workspace=h_ws, out=h_out, device=dev, stream=stream)

    e2e_step()
    torch.cuda.synchronize()
    assert torch.equal(h_out["iters"], out["iters"].cpu()), "host pipeline differs from the device solve"
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    ems, _ = reduce_metric(e0.elapsed_time(e1), vox_iters, dev)
    e2e_value = work_all / (ems / args.steps / 1000.0)
    h2d = h_vol.numel() * h_vol.element_size() + h_fixed.numel() + h_values.numel() * 4
    d2h = h_out["labels"].numel() + BATCH * 12
    del h_ws

    # ---------------- rows a8 / a9 beside the headline (not part of the step) ----------------
    rows = None if (args.no_rows or rank != 0) else pyramid_and_queue(dev)

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, dt, vi, cores = cpu_oracle_sample(args.cpu_bricks)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{args.cpu_bricks} cfg2 bricks (64^3) at rel tol 1e-6, {dt:.1f}s, "
                         "fp64 numpy/scipy CSR Jacobi-PCG, 1 thread"}
    gpu_launches = sum(launches.values())
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "batch_per_gpu": BATCH, "brick": [N, N, N],
                   "global_batch": BATCH * world, "parallelism": f"bricks sharded over {world} GPU(s), no collective",
                   "l2": "inputs larger than L2 (u16 volume, mask, values, weight planes, CG state: > 2 GB), no flush",
                   "iters": {"min": int(iters.min()), "median": float(np.median(iters)),
                             "max": int(iters.max())}},
        "bricks_per_s": BATCH * world / (ms_per_step / 1000.0),
        "full_solve_ms": ms_per_step,
        "solver": solver_used,
        "roofline": roofline,
        "streaming": streaming,
        "pyramid_queue": rows,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": ems / args.steps,
                "api": "rw_solve_bricks_host (pinned host buffers, chunked H2D/solve/D2H overlap)",
                "chunk": args.e2e_chunk or -(-BATCH // 32)},
        "gpu_launches": int(gpu_launches),
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--e2e-chunk", type=int, default=0,
                    help="bricks per pipeline chunk of the e2e host-buffer solve (0: batch/32)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workers", type=int, default=min(16, os.cpu_count() or 1))
    ap.add_argument("--cpu-bricks", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solver", default="auto", choices=["auto", "streaming", "resident"])
    ap.add_argument("--no-streaming", action="store_true",
                    help="skip the secondary streaming-solver timing")
    ap.add_argument("--no-rows", action="store_true",
                    help="skip the secondary pyramid / queue measurements")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
