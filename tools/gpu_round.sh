# One gpurun call: GPU tests, smoke, bench (with cpu_baseline), per-config lines,
# ncu launch list of the bench command, ncu --set full of the resident kernel.
# Usage: gpurun -- 'bash tools/gpu_round.sh TAG'   (SKIP_TESTS=1 / SKIP_CFGS=1 to skip)
cd $GRAFT_REPO_ROOT
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
if [ "${SKIP_TESTS:-0}" = "0" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"
tail -3 $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json; tail -3 $O/bench.err
if [ "${SKIP_CFGS:-0}" = "0" ]; then
timeout 1200 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"
cat $O/configs.jsonl; tail -3 $O/configs.err
fi
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-streaming --no-rows"
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv $CMD > $O/ncu1.log 2>&1; echo "ncu1 rc=$?"
if [ "${SKIP_FULL:-0}" = "0" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resident -s 3 -c 1 -o $O/resident $CMD > $O/ncu2.log 2>&1; echo "ncu2 rc=$?"
# the streaming solver's dominant kernel (one-pass pass A) at a steady-state iteration
SCMD="python bench.py --solver streaming --host-loop --steps 1 --warmup 3 --no-cpu-baseline --no-rows --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 60 -c 1 -o $O/passA $SCMD > $O/ncu3.log 2>&1; echo "ncu3 rc=$?"
fi
# summaries on the box (gpurun copies back at most 64 MiB): the .ncu-rep files are dropped
# unless KEEP_REP=1
if [ "${SKIP_FULL:-0}" = "0" ]; then
python tools/ncu_summary.py --launches $O/launches.csv --rep $O/resident.ncu-rep $O/passA.ncu-rep --bench $O/bench.json --out $O/summary > /dev/null 2>&1; echo "summary rc=$?"
timeout 300 python tools/ncu_hot.py $O/resident.ncu-rep 40 > $O/resident_hot.txt 2>&1
timeout 300 python tools/ncu_hot.py $O/passA.ncu-rep 40 > $O/passA_hot.txt 2>&1
[ "${KEEP_REP:-0}" = "1" ] || rm -f $O/*.ncu-rep
fi
ls -la $O
