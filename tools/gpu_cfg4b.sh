cd $GRAFT_REPO_ROOT
O=gpurun_out/c4b; mkdir -p $O
timeout 900 python tools/lastdec_ab.py ns > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?"; cat $O/ab.jsonl; tail -2 $O/ab.err
timeout 900 python tools/zc_sweep.py 0 32 > $O/sweep.jsonl 2> $O/sweep.err; echo "sweep rc=$?"; cat $O/sweep.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_hier.py -q -x --timeout 600 2>&1 | tail -3
