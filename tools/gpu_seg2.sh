# cfg3 tile-shape A/B: head library vs current (loop restructure), TY / ZC wave balancing
cd $GRAFT_REPO_ROOT
O=gpurun_out/seg2; mkdir -p $O
for i in 1 2; do
RW_LIB_PATH=abtest/librw_head.so timeout 300 python tools/cfg3_sweep.py 300 0:16 > $O/head_$i.jsonl 2>&1; echo head; cat $O/head_$i.jsonl
RW_PASSA_SEG=0 timeout 300 python tools/cfg3_sweep.py 300 0:16 > $O/new_$i.jsonl 2>&1; echo new; cat $O/new_$i.jsonl
done
for ty in 14 15; do
RW_PASSA_SEG=0 RW_TY=$ty timeout 300 python tools/cfg3_sweep.py 300 256:16 128:16 0:16 > $O/ty$ty.jsonl 2>&1; echo "ty=$ty (zc 256,128,64)"; cat $O/ty$ty.jsonl
done
RW_PASSA_SEG=0 timeout 300 python tools/cfg3_sweep.py 300 256:16 128:16 > $O/ty16.jsonl 2>&1; echo "ty=16 (zc 256,128)"; cat $O/ty16.jsonl
