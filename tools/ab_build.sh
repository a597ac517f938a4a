# build abtest/librw_{old,new}.so (+ timing variants t*) : old = resident.cu at git HEAD
# (or $OLD_REV), new = the working tree
set -e
cd /root/repo
mkdir -p abtest
F=paper_2103_09564_b200/csrc/resident.cu
cp $F /tmp/res_new.cu
git show ${OLD_REV:-HEAD}:$F > /tmp/res_old.cu
cp /tmp/res_old.cu $F
RW_NVCC_DEFS="$DEFS" python -m paper_2103_09564_b200.build --out abtest/librw_old.so > /dev/null
RW_NVCC_DEFS="$DEFS -DRW_RES_TIMING" python -m paper_2103_09564_b200.build --out abtest/librw_told.so > /dev/null
cp /tmp/res_new.cu $F
RW_NVCC_DEFS="$DEFS" python -m paper_2103_09564_b200.build --out abtest/librw_new.so > /dev/null
RW_NVCC_DEFS="$DEFS -DRW_RES_TIMING" python -m paper_2103_09564_b200.build --out abtest/librw_tnew.so > /dev/null
python -m paper_2103_09564_b200.build > /dev/null
echo built
