cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/res1
timeout 600 python -m pytest tests/test_gpu_resident.py -x -q --timeout 300 > gpurun_out/res1/tests.log 2>&1; echo "res tests rc=$?"; tail -30 gpurun_out/res1/tests.log
timeout 300 python tools/res_time.py 64 2>&1 | tail -5
