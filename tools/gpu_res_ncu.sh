cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/resncu
python tools/res_time.py 64 > gpurun_out/resncu/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o gpurun_out/resncu/res python tools/res_time.py 64 > gpurun_out/resncu/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/resncu/ncu.log
