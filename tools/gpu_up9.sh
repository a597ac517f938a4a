# k_upsample quad order A/B (RW_UPSAMPLE_V=0 round robin, 1 column walk) on the cfg5 2048^3
# hierarchical run + the hierarchical GPU tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/upcol
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_hier.py tests/test_gpu_hier_ooc.py -m gpu -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for v in 0 1; do
  RW_UPSAMPLE_V=$v timeout 600 python tools/bench_hier.py --scale 1.0 > $O/hier_v${v}.jsonl 2> $O/hier_v${v}.err; echo "v=$v rc=$?"
  python - <<PY
import json
for l in open("$O/hier_v${v}.jsonl"):
    d = json.loads(l)
    print("v=$v", d.get("config","")[-40:], round(d.get("ms",0),2), d.get("kernel_ms_all_reps",{}).get("hier"))
PY
done
