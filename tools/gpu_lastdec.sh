cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ld
RW_LASTDEC_MIN_U=100000000 timeout 600 python tools/lastdec_ab.py off > gpurun_out/ld/ab.jsonl 2> gpurun_out/ld/off.err; echo "off rc=$?"
timeout 600 python tools/lastdec_ab.py on >> gpurun_out/ld/ab.jsonl 2> gpurun_out/ld/on.err; echo "on rc=$?"
cat gpurun_out/ld/ab.jsonl; tail -3 gpurun_out/ld/*.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 600 2>&1 | tail -3
