cd $GRAFT_REPO_ROOT
O=gpurun_out/c34; mkdir -p $O
python tools/prof_cfg3.py > $O/plain3.log 2>&1; echo "plain3 rc=$?"; cat $O/plain3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 12 -c 1 -o $O/cfg3_passA python tools/prof_cfg3.py > $O/ncu3.log 2>&1; echo "ncu3 rc=$?"
python tools/prof_cfg4.py > $O/plain4.log 2>&1; echo "plain4 rc=$?"; cat $O/plain4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 12 -c 1 -o $O/cfg4_passA python tools/prof_cfg4.py > $O/ncu4.log 2>&1; echo "ncu4 rc=$?"
