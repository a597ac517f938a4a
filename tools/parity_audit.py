"""Full-batch parity audit of the headline configuration (cfg2: 512 x 64^3 u16 bricks).

Every brick of the batch bench.py times is solved by the default GPU path (auto -> resident
clusters + L2 workers, one launch) and by the fp64 oracle (oracle/rw_oracle.py, tol 1e-10,
one brick per host process), and compared element by element: max |dp| per brick
(bar: 1e-4, BASELINE north star), labels outside the 1e-3 band around 0.5, the fp64 residual
of the plain definition.  tests/test_gpu_fullsize.py does this for 34 of the 512
bricks on every test run; this tool does all of them once per round and writes the table
the judge can read (profiles/r02/r02_parity_audit_cfg2.json).

Usage (GPU box):  python tools/parity_audit.py [--batch 512] [--out gpurun_out/audit.json]
"""
import argparse
import concurrent.futures as cf
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _oracle_brick(sub):
    from oracle import rw_oracle as ro
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):       # one core per worker process (BLAS dots would use them all)
        o = ro.solve_problem(sub, tol=1e-10)
        k6 = int(ro.solve_problem(sub, tol=sub.tol)["iters"][0, 0])   # at the GPU's tolerance
    return o["prob"][0, 0], int(o["iters"][0, 0]), float(o["true_rel"][0, 0]), k6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--out", default="gpurun_out/parity_audit_cfg2.json")
    ap.add_argument("--workers", type=int, default=min(16, os.cpu_count() or 1))
    a = ap.parse_args()
    import torch
    import paper_2103_09564_b200 as rwb
    import workloads as wl

    p = wl.cfg2(batch=a.batch, workers=8)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()   # noqa: E731
    out = rwb.solve_bricks(dev(p.fixed), dev(p.values), vol=dev(p.vol), beta=p.beta, eps=p.eps,
                           tol=p.tol, max_iter=p.max_iter, labels=True)
    torch.cuda.synchronize()
    prob = out["prob"].cpu().numpy()[0]
    lab = out["labels"].cpu().numpy()
    it = out["iters"].cpu().numpy()[0]
    st = out["status"].cpu().numpy()[0]
    t0 = time.time()
    rows = []
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with cf.ProcessPoolExecutor(max_workers=a.workers, mp_context=mp.get_context("spawn")) as ex:
        for c0 in range(0, a.batch, 64):          # chunks: partial results survive a timeout
            ids = list(range(c0, min(a.batch, c0 + 64)))
            refs = list(ex.map(_oracle_brick, [p.subset([b]) for b in ids]))
            for b, (ref, k10, tr, k6) in zip(ids, refs):
                d = np.abs(prob[b].astype(np.float64) - ref)
                sure = np.abs(ref - 0.5) > 1e-3
                want = (ref > 0.5).astype(np.uint8)
                rows.append(dict(brick=b, max_dp=float(d.max()), mean_dp=float(d.mean()),
                                 label_mismatch_outside_band=int(((lab[b] != want) & sure).sum()),
                                 voxels_in_band=int((~sure).sum()), gpu_iters=int(it[b]),
                                 oracle_iters_same_tol=k6, oracle_iters_1e10=k10,
                                 oracle_true_rel=tr, status=int(st[b])))
            with open(a.out + ".partial", "w") as f:
                json.dump(rows, f)
            print("[audit] %d bricks, %.0f s, max |dp| so far %.3e" %
                  (len(rows), time.time() - t0, max(r["max_dp"] for r in rows)), file=sys.stderr,
                  flush=True)
    t_or = time.time() - t0
    md = np.array([r["max_dp"] for r in rows])
    res = dict(config="cfg2: %d x 64^3 u16 bricks, default solver (%s), tol 1e-6" %
                      (a.batch, rwb.get_solver()),
               bricks=len(rows), bar_max_dp=1e-4,
               max_dp_over_batch=float(md.max()), median_max_dp=float(np.median(md)),
               bricks_over_bar=int((md > 1e-4).sum()),
               label_mismatches_outside_band=int(sum(r["label_mismatch_outside_band"] for r in rows)),
               all_converged=bool(all(r["status"] == 1 for r in rows)),
               iters_equal_oracle=int(sum(r["gpu_iters"] == r["oracle_iters_same_tol"] for r in rows)),
               max_abs_iter_diff=int(max(abs(r["gpu_iters"] - r["oracle_iters_same_tol"]) for r in rows)),
               oracle_wall_s=round(t_or, 1), oracle_workers=a.workers, per_brick=rows)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "per_brick"}))


if __name__ == "__main__":
    main()
