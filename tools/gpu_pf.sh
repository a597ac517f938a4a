cd $GRAFT_REPO_ROOT
O=gpurun_out/pf; mkdir -p $O
for pf in 0 2 4 0 2 4; do RW_PASSA_PF=$pf timeout 600 python tools/lastdec_ab.py pf$pf >> $O/ab.jsonl 2> $O/pf$pf.err; echo "pf$pf rc=$?"; done
cat $O/ab.jsonl
for pf in 0 2 4; do RW_PASSA_PF=$pf timeout 300 python bench.py --solver streaming --steps 3 --warmup 3 --no-cpu-baseline --no-rows --no-configs 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf$pf cfg2-streaming', d['value']/1e9, d['ms_per_step'])"; done
