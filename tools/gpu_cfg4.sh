cd $GRAFT_REPO_ROOT
O=gpurun_out/c4; mkdir -p $O
timeout 900 python tools/zc_sweep.py 0 32 16 > $O/sweep.jsonl 2> $O/sweep.err; echo "sweep rc=$?"; cat $O/sweep.jsonl
python tools/prof_cfg4.py > $O/plain.log 2>&1; echo "plain rc=$?"; cat $O/plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 12 -c 1 -o $O/cfg4_passA python tools/prof_cfg4.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
