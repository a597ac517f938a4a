cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/rc
for rc in 0 1 3; do RW_PASSA_RC=$rc timeout 600 python tools/lastdec_ab.py rc$rc >> gpurun_out/rc/ab.jsonl 2> gpurun_out/rc/rc$rc.err; echo "rc$rc rc=$?"; done
cat gpurun_out/rc/ab.jsonl
