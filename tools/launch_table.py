"""Aggregate an ncu --csv launch list (time + DRAM bytes) per kernel: python tools/launch_table.py file.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
K, M, V, U = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
T = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= V:
        continue
    name = r[K].split("(")[0].replace("void ", "")
    v = float(r[V].replace(",", ""))
    if r[M] == "gpu__time_duration.sum":
        cnt[name] += 1
        agg[name]["ms"] += v * T.get(r[U], 1.0)
    else:
        agg[name]["GB"] += v * B.get(r[U], 1.0) / 1e9
for n, d in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
    print(f"{n:42s} n={cnt[n]:5d} ms={d['ms']:10.2f} GB={d['GB']:9.2f} GB/s={d['GB'] / (d['ms'] / 1e3) if d['ms'] else 0:8.0f}")
