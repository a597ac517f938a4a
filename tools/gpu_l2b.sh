cd $GRAFT_REPO_ROOT
O=gpurun_out/l2b; mkdir -p $O
RW_DEBUG_L2W=1 timeout 900 python tools/l2w_ab.py 512 0 16 32 48 64 96 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?"
cat $O/ab.jsonl; grep "\[l2w\]" $O/ab.err | sort | uniq -c
