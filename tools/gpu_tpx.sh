cd $GRAFT_REPO_ROOT
O=gpurun_out/tpx; mkdir -p $O
for t in 16 32 64; do RW_TPX=$t timeout 600 python tools/lastdec_ab.py tpx$t >> $O/ab.jsonl 2> $O/t$t.err; echo "tpx$t rc=$?"; done
cat $O/ab.jsonl
