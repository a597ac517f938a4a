cd $GRAFT_REPO_ROOT
O=gpurun_out/host1; mkdir -p $O
timeout 600 python tools/host_ab.py 512 0 8 32 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?"; cat $O/ab.jsonl; tail -5 $O/ab.err
timeout 900 python -m pytest tests/test_gpu_host.py tests/test_gpu_resident.py -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -5 $O/tests.log
