"""Attribute ncu per-SASS stall samples to (outermost) source lines of one kernel.
usage: ncu_lines.py <sass-page.csv> <nvdisasm -gi listing> <function substring> <src substring>
The listing must come from the same cubin as the profiled kernel (offsets match)."""
import csv, re, sys, collections
csvp, lst, fn, src = sys.argv[1:5]
r = list(csv.reader(open(csvp)))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:]]
base = int(rows[0]["Address"], 16)
# offset -> line
line_of = {}
inside, cur = False, None
for L in open(lst):
    if L.startswith("//--------------------- .text."):
        inside = fn in L
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', L)
    if m:
        if src in m.group(1):
            cur = int(m.group(2))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", L)
    if m:
        line_of[int(m.group(1), 16)] = (cur, m.group(2).split(";")[0].strip())
keys = ["stall_short_sb", "stall_barrier", "stall_not_selected", "stall_selected", "stall_wait",
        "stall_long_sb", "stall_mio", "stall_dispatch", "stall_math", "stall_branch_resolving", "stall_lg", "stall_membar"]
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
mism = 0
for d in rows:
    off = int(d["Address"], 16) - base
    ln, ins = line_of.get(off, (None, "?"))
    sass = d["Source"].strip().split(";")[0].strip()
    if ins != "?" and ins.split()[0] != sass.split()[0]:
        mism += 1
    for k in keys + ["Warp Stall Sampling (All Samples)"]:
        v = d.get(k, "0") or "0"
        agg[ln][k] += int(float(v))
        tot[k] += int(float(v))
    agg[ln]["inst"] += int(d.get("Instructions Executed", "0") or 0)
print("opcode mismatches:", mism, "of", len(rows))
T = tot["Warp Stall Sampling (All Samples)"]
print("total samples", T, {k[6:]: round(tot[k] / T * 100, 1) for k in keys})
for ln in sorted(agg, key=lambda l: -agg[l]["Warp Stall Sampling (All Samples)"])[:int(sys.argv[5]) if len(sys.argv) > 5 else 30]:
    a = agg[ln]
    s = a["Warp Stall Sampling (All Samples)"]
    top = sorted(((a[k], k[6:]) for k in keys), reverse=True)[:4]
    print(f"line {ln}: {s / T * 100:5.1f}%  inst {a['inst']:>10d}  " + " ".join(f"{n}={v / T * 100:.1f}" for v, n in top))
