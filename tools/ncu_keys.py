"""Print selected raw metrics of every kernel in an ncu report (run on the GPU box).
    python tools/ncu_keys.py report.ncu-rep [substring ...]"""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
rep = sys.argv[1]
subs = sys.argv[2:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, rows = r[0], r[1], r[2:]
for row in rows:
    d = dict(zip(h, row))
    u = dict(zip(h, units))
    print("==", d.get("Kernel Name", "?")[:120])
    for k in KEYS + [k for k in h if any(s in k for s in subs)]:
        if k in d:
            print(f"  {k} = {d[k]} {u.get(k, '')}")
    st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
    for k, v in sorted(st, key=lambda x: -x[1])[:10]:
        print(f"  stall {v:7.3f} {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}")
