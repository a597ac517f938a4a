"""Hot SASS lines + stall summary of one kernel in an ncu report.
    python tools/ncu_hot.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, rows = r[0], r[2:]
for row in rows[:1]:
    d = dict(zip(h, row))
    for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__cycles_active.avg",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"):
        print(k, d.get(k))
    st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
    for k, v in sorted(st, key=lambda x: -x[1])[:12]:
        print(f"  {v:7.3f} {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h = r[1]
data = [dict(zip(h, x)) for x in r[2:]]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("samples", tot, "sass lines", len(data))
idx = sorted(range(len(data)), key=lambda i: -int(data[i]["Warp Stall Sampling (All Samples)"] or 0))
for i in idx[:top]:
    d = data[i]
    print(f"{i:5d} {int(d['Warp Stall Sampling (All Samples)'])/tot*100:5.1f}% {d['Source'][:90]}")
