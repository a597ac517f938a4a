# A/B: head library vs current build on cfg3 (300 iterations) and cfg2 streaming (512 bricks)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab3; mkdir -p $O
for i in 1 2; do
for L in abtest/librw_head.so paper_2103_09564_b200/librw.so; do
RW_LIB_PATH=$L timeout 300 python tools/cfg3_sweep.py 300 0:16 > $O/c3.jsonl 2>&1; echo "$L cfg3 $(cat $O/c3.jsonl | cut -c1-120)"
RW_LIB_PATH=$L timeout 300 python tools/stream_time.py 512 > $O/c2.jsonl 2>&1; echo "$L cfg2s $(cat $O/c2.jsonl | cut -c1-100)"
done; done
