cd $GRAFT_REPO_ROOT
T=${TAG:-bench}
timeout 900 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} > gpurun_out/$T.json 2> gpurun_out/$T.err; echo "bench rc=$?"
tail -3 gpurun_out/$T.err
