# pass-A segments: parity tests + cfg3 / cfg4 A/B (RW_PASSA_SEG 0 vs 1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/seg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for s in 0 1 0 1; do
RW_PASSA_SEG=$s timeout 300 python tools/cfg3_sweep.py 300 0:16 > $O/cfg3_$s.jsonl 2>&1; echo "seg=$s"; cat $O/cfg3_$s.jsonl
done
for s in 0 1; do
RW_PASSA_SEG=$s timeout 600 python tools/bench_configs.py > $O/cfg_$s.jsonl 2> $O/cfg_$s.err; echo "configs seg=$s rc=$?"; grep -E "cfg3|cfg4" $O/cfg_$s.jsonl
done
