# A/B of resident-kernel variants built into abtest/ (librw_<v>.so and timing builds
# librw_t<v>.so): correctness + throughput on 512 cfg2 bricks, phase cycles on 64
cd $GRAFT_REPO_ROOT
O=gpurun_out/${AB_TAG:-ab}
mkdir -p $O
for v in ${AB_VARIANTS:-old new}; do
  RES_DUMP=/tmp/ab_$v.npz RW_LIB_PATH=$PWD/abtest/librw_$v.so timeout 300 python tools/res_time.py 512 > $O/$v.log 2>&1
  echo "== $v rc=$?"; grep -E '"resident"|max_abs' $O/$v.log | cut -c1-200
  RW_LIB_PATH=$PWD/abtest/librw_t$v.so RW_DEBUG_RES_TIMING=1 timeout 300 python tools/res_time.py 64 > $O/t$v.log 2>&1
  grep "res-timing" $O/t$v.log | head -4
done
python - <<'PY'
import numpy as np, os
vs = os.environ.get("AB_VARIANTS", "old new").split()
ref = np.load(f"/tmp/ab_{vs[0]}.npz")
for v in vs[1:]:
    o = np.load(f"/tmp/ab_{v}.npz")
    print(v, "vs", vs[0], "prob bitwise equal:", np.array_equal(o["prob"], ref["prob"]),
          "max|dp|:", float(np.abs(o["prob"] - ref["prob"]).max()), "iters equal:", np.array_equal(o["it"], ref["it"]))
PY
