cd $GRAFT_REPO_ROOT
O=gpurun_out/seg; mkdir -p $O
for sg in 0 -1 0 -1; do RW_PASSA_SEG=$sg timeout 600 python tools/lastdec_ab.py seg$sg >> $O/ab.jsonl 2> $O/seg$sg.err; echo "seg$sg rc=$?"; tail -2 $O/seg$sg.err; done
cat $O/ab.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_hier.py tests/test_gpu_weights_ex.py -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
