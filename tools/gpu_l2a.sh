cd $GRAFT_REPO_ROOT
O=gpurun_out/l2a; mkdir -p $O
cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mb_cores mb_cores.cu && timeout 120 ./mb_cores > ../../$O/cores.jsonl 2>&1; echo "cores rc=$?"; cd ../..
cat $O/cores.jsonl
timeout 600 python tools/l2only.py 128 9 18 37 > $O/l2only.jsonl 2> $O/l2only.err; echo "l2only rc=$?"
cat $O/l2only.jsonl; tail -3 $O/l2only.err
RW_L2_ONLY=1 RW_L2_NW=9 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l2res -s 4 -c 1 -o $O/l2res python tools/l2only.py 64 9 > $O/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 $O/ncu.log
