cd $GRAFT_REPO_ROOT
O=gpurun_out/l2c; mkdir -p $O
export RW_DEBUG_L2W=1
for v in base cs evl both base; do
  if [ $v = base ]; then L=$PWD/paper_2103_09564_b200/librw.so; else L=$PWD/abtest/librw_$v.so; fi
  RW_LIB_PATH=$L timeout 300 python tools/l2w_ab.py 512 48 > $O/ab_$v.jsonl 2> $O/ab_$v.err; echo "$v rc=$?"
  tail -1 $O/ab_$v.jsonl; grep "\[l2w\]" $O/ab_$v.err | tail -2
done
unset RW_DEBUG_L2W
timeout 300 python tools/l2only.py 128 9 > $O/iso.jsonl 2>&1; echo "iso rc=$?"; tail -1 $O/iso.jsonl
RW_L2_HOLD=1 timeout 300 python tools/l2only.py 128 9 > $O/hold.jsonl 2>&1; echo "hold rc=$?"; tail -1 $O/hold.jsonl
RW_LIB_PATH=$PWD/abtest/librw_evl.so RW_L2_HOLD=1 timeout 300 python tools/l2only.py 128 9 > $O/hold_evl.jsonl 2>&1; echo "hold_evl rc=$?"; tail -1 $O/hold_evl.jsonl
