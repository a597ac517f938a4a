# One gpurun call: GPU tests, smoke, bench (with cpu_baseline), per-config lines,
# ncu launch list of the bench command.  Usage: gpurun -- 'bash tools/gpu_round.sh TAG'
cd $GRAFT_REPO_ROOT
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"
tail -3 $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json; tail -3 $O/bench.err
if [ "${SKIP_CFGS:-0}" = "0" ]; then
timeout 1200 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"
cat $O/configs.jsonl; tail -3 $O/configs.err
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu1.log 2>&1; echo "ncu1 rc=$?"
ls -la $O
