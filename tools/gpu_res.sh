# resident-solver iteration: tests + timing (+ optional ncu with NCU=1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-res}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_resident.py -x -q --timeout 300 > $O/tests.log 2>&1; echo "res tests rc=$?"; tail -15 $O/tests.log
timeout 300 python tools/res_time.py ${NB:-64} > $O/time.log 2>&1; echo "time rc=$?"; tail -4 $O/time.log
if [ "${NCU:-0}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o $O/res python tools/res_time.py 64 > $O/ncu.log 2>&1; echo "ncu rc=$?"
fi
