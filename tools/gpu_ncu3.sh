cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu3; mkdir -p $O
python tools/prof_passA1.py 1 > $O/plain.log 2>&1; echo "plain rc=$?"; cat $O/plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 12 -c 1 -o $O/cfg3_passA python tools/prof_passA1.py 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
SCMD="python bench.py --solver streaming --host-loop --steps 1 --warmup 3 --no-cpu-baseline --no-rows --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 60 -c 1 -o $O/cfg2_passA $SCMD > $O/ncu2.log 2>&1; echo "ncu2 rc=$?"
ls -la $O
