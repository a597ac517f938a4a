cd $GRAFT_REPO_ROOT
O=gpurun_out/il; mkdir -p $O
for v in il0 il1 il0 il1; do RW_LIB_PATH=$PWD/abtest/librw_$v.so timeout 600 python tools/lastdec_ab.py $v >> $O/ab.jsonl 2> $O/$v.err; echo "$v rc=$?"; done
cat $O/ab.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "label or rhs or multi" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
