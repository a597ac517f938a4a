cd $GRAFT_REPO_ROOT
O=gpurun_out/w2; mkdir -p $O
RW_DEBUG_L2W=1 timeout 300 python tools/l2w_ab.py 512 48 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?"; cat $O/ab.jsonl; grep "\[l2w\]" $O/ab.err | sort | uniq -c
RW_L2_HOLD=1 timeout 300 python tools/l2only.py 128 9 > $O/hold.jsonl 2>&1; echo "hold rc=$?"; tail -1 $O/hold.jsonl
timeout 300 python tools/host_ab.py 512 0 > $O/host.jsonl 2>&1; echo "host rc=$?"; head -1 $O/host.jsonl
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_host.py tests/test_gpu_fullsize.py -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-streaming --no-rows --no-configs"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv $CMD > $O/ncu1.log 2>&1; echo "ncu1 rc=$?"; tail -2 $O/ncu1.log
