# k_upsample vs k_upsample9 (RW_UPSAMPLE_V) on the cfg5 2048^3 hierarchical run, the
# hierarchical GPU tests (bit-identity of the in-HBM field with the OOC driver / oracle parity),
# then the all-brick cfg2 parity audit.
cd $GRAFT_REPO_ROOT
O=gpurun_out/up9
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_hier.py tests/test_gpu_hier_ooc.py -m gpu -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for v in 0 9 0 9; do
  RW_UPSAMPLE_V=$v timeout 600 python tools/bench_hier.py --scale 1.0 > $O/hier_v${v}.jsonl 2> $O/hier_v${v}.err; echo "v=$v rc=$?"
  python - <<PY
import json
for l in open("$O/hier_v${v}.jsonl"):
    d = json.loads(l)
    print("v=$v", d.get("config","")[-40:], round(d.get("ms",0),2), d.get("kernel_ms_all_reps",{}).get("hier"))
PY
done
timeout 1500 python tools/parity_audit.py --out $O/parity_audit_cfg2.json 2> $O/audit.err | cut -c1-900; tail -3 $O/audit.err
