cd $GRAFT_REPO_ROOT
tools/micro/mb_graphwhile
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "device_loop" --timeout 300 2>&1 | tail -5
timeout 900 python tools/devloop_ab.py > gpurun_out/r2d_devloop.jsonl 2> gpurun_out/r2d_devloop.err; echo "ab rc=$?"
cat gpurun_out/r2d_devloop.jsonl; tail -3 gpurun_out/r2d_devloop.err
