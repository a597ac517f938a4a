# ncu --set full of the 2048^3 upsample launch of one cfg5 H_p run (the 6th upsample launch)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_up
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_hier_ooc.py -m gpu -q -x --timeout 300 -k bitwise > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_upsample -s 5 -c 1 -o $O/up python tools/bench_hier.py --scale 1.0 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_keys.py $O/up.ncu-rep l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit > $O/keys.txt 2>&1
timeout 300 python tools/ncu_hot.py $O/up.ncu-rep 30 > $O/hot.txt 2>&1
rm -f $O/*.ncu-rep
cat $O/keys.txt | head -40; head -40 $O/hot.txt
