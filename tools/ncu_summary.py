#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/pass.ncu-rep --bench gpurun_out/bench.json --out profiles/r01_v1

Writes <out>.md (human summary) and <out>.json; also updates profiles/ncu_traffic.json
(per-launch DRAM bytes of each captured kernel, read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

UNITS = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
       "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
       "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__t_bytes.sum", "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic"]


def short(name):
    return name.split("(")[0].replace("void ", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        tot[short(r[ki])] += v
        cnt[short(r[ki])] += 1
    T = sum(tot.values())
    return {k: {"launches": cnt[k], "ms": tot[k], "share": tot[k] / T} for k in
            sorted(tot, key=lambda k: -tot[k])}


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m in RAW:
            if m in h:
                i = h.index(m)
                val = r[i].replace(",", "")
                try:
                    v = float(val)
                except ValueError:
                    continue
                u = units[i]
                if u in BYTES:
                    v *= BYTES[u]
                    u = "byte"
                if u in UNITS:
                    v *= UNITS[u]
                    u = "ms"
                d[m] = v
        if "dram__bytes_read.sum" in d:
            d["dram_bytes"] = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0)
            d["dram_GBps"] = d["dram_bytes"] / (d["gpu__time_duration.sum"] * 1e-3) / 1e9
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--bench")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    S = {"note": a.note}
    md = [f"# ncu summary {os.path.basename(a.out)}", "", a.note, ""]
    if a.bench and os.path.exists(a.bench):
        b = json.loads(open(a.bench).read().strip().splitlines()[-1])
        S["bench"] = b
        md += ["## bench.py line", "", "```", json.dumps(b, indent=1)[:4000], "```", ""]
    if a.launches:
        L = launches(a.launches)
        S["launch_list"] = L
        md += ["## launch list (ncu --metrics gpu__time_duration.sum, cold/serialised)", "",
               "| kernel | launches | ms | share |", "|---|---|---|---|"]
        md += [f"| {k} | {v['launches']} | {v['ms']:.3f} | {v['share']:.3f} |" for k, v in L.items()]
        md.append("")
    if a.rep:
        R = [d for r_ in a.rep for d in rep(r_)]
        S["full_capture"] = R
        md += ["## ncu --set full (one launch each, all bricks active)", ""]
        for d in R:
            md.append(f"### {d['kernel']}")
            md += [f"- {k}: {v:.6g}" if isinstance(v, float) else f"- {k}: {v}" for k, v in d.items() if k != "kernel"]
            md.append("")
        tp = os.path.join(os.path.dirname(a.out), "ncu_traffic.json")
        T = json.load(open(tp)) if os.path.exists(tp) else {}
        for d in R:
            key = {"k_passA": "passA", "k_passB": "passB", "k_resident": "resident"}.get(
                d["kernel"].split("<")[0], d["kernel"])
            if "dram_bytes" in d:
                T[key] = d["dram_bytes"]
        T["_source"] = os.path.basename(a.out)
        json.dump(T, open(tp, "w"), indent=1)
    json.dump(S, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".md", "w").write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
