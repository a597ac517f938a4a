cd $GRAFT_REPO_ROOT
O=gpurun_out/abring; mkdir -p $O
for v in old new old new; do
  RW_LIB_PATH=$PWD/abtest/librw_$v.so timeout 300 python tools/l2w_ab.py 512 48 > $O/ab_$v.jsonl 2>/dev/null; echo "$v: $(tail -2 $O/ab_$v.jsonl | python -c 'import sys,json; print([ (json.loads(l)["workers"], round(json.loads(l)["ms"],2)) for l in sys.stdin])')"
done
