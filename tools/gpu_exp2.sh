cd $GRAFT_REPO_ROOT
O=gpurun_out/exp2; mkdir -p $O
python tools/prof_cfg3.py > $O/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 12 -c 1 -o $O/c3 python tools/prof_cfg3.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_keys.py $O/c3.ncu-rep > $O/c3_keys.txt 2>&1
timeout 300 python tools/ncu_hot.py $O/c3.ncu-rep 40 > $O/c3_hot.txt 2>&1
SCMD="python bench.py --solver streaming --host-loop --steps 1 --warmup 3 --no-cpu-baseline --no-rows --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_passA -s 60 -c 1 -o $O/c2 $SCMD > $O/ncu2.log 2>&1; echo "ncu2 rc=$?"
python tools/ncu_keys.py $O/c2.ncu-rep > $O/c2_keys.txt 2>&1
rm -f $O/*.ncu-rep
