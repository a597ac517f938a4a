cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/r2a_tests.log 2>&1
echo "tests rc=$?"
tail -5 gpurun_out/r2a_tests.log
timeout 300 python tools/cosched_sweep.py 0 100 150 200 250 300 > gpurun_out/r2a_cosched.jsonl 2>&1; echo "cosched rc=$?"
cat gpurun_out/r2a_cosched.jsonl
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
