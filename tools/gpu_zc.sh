cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/zc
timeout 1200 python tools/zc_sweep.py ${ZCS:-0 48 32 24 16} > gpurun_out/zc/sweep.jsonl 2> gpurun_out/zc/sweep.err; echo "sweep rc=$?"
cat gpurun_out/zc/sweep.jsonl; tail -3 gpurun_out/zc/sweep.err
