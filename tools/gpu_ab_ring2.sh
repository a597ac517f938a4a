cd $GRAFT_REPO_ROOT
O=gpurun_out/abring2; mkdir -p $O
for v in old new old new; do
  RW_LIB_PATH=$PWD/abtest/librw_$v.so timeout 300 python tools/l2w_ab.py 512 48 > $O/ab_$v.jsonl 2>/dev/null; echo "$v: $(tail -2 $O/ab_$v.jsonl | python -c 'import sys,json; print([ (json.loads(l)["workers"], round(json.loads(l)["ms"],2), json.loads(l).get("bitwise_equal")) for l in sys.stdin])')"
done
timeout 300 python tools/host_ab.py 512 0 > $O/host.jsonl 2>&1; echo "host rc=$?"; head -1 $O/host.jsonl
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_host.py -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
