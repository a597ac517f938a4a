# experiment call: cfg3 z-chunk / tile sweep; cosched re-measurement after the fork fix
cd $GRAFT_REPO_ROOT
O=gpurun_out/exp1; mkdir -p $O
timeout 600 python tools/cfg3_sweep.py 300 0:16 32:16 37:16 43:16 52:16 16:16 0:8 0:32 > $O/cfg3.jsonl 2> $O/cfg3.err; echo "cfg3 rc=$?"
cat $O/cfg3.jsonl; tail -3 $O/cfg3.err
RW_OPT=1 timeout 600 python tools/cosched_sweep.py 0 40 80 120 200 > $O/cosched.jsonl 2> $O/cosched.err; echo "cosched rc=$?"
cat $O/cosched.jsonl; tail -3 $O/cosched.err
