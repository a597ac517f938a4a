# A/B of abtest/librw_{old,new}.so on tools/res_n.py (brick side N, batch B)
cd $GRAFT_REPO_ROOT
RW_LIB_PATH=$PWD/abtest/librw_old.so timeout 300 python tools/res_n.py ${N:-40} ${B:-1024} > /dev/null 2>&1   # clocks up
for v in old new old new; do
  RES_DUMP=/tmp/abn_$v.npz RW_LIB_PATH=$PWD/abtest/librw_$v.so timeout 300 python tools/res_n.py ${N:-40} ${B:-1024}
done
python -c "
import numpy as np
a=np.load('/tmp/abn_old.npz'); b=np.load('/tmp/abn_new.npz')
print('prob equal', np.array_equal(a['prob'],b['prob']), 'max dp', float(np.abs(a['prob']-b['prob']).max()), 'iters equal', np.array_equal(a['it'],b['it']))"
