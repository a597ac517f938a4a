# A/B of streaming builds: abtest/librw_head.so vs the in-tree build (timings + output hashes)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab4; mkdir -p $O
for i in 1 2; do
for L in abtest/librw_head.so paper_2103_09564_b200/librw.so; do
echo "== $L"; RW_LIB_PATH=$L timeout 600 python tools/stream_ab.py ${CASES:-cfg3,cfg2,cfg4} 2>&1 | tail -4
done; done
