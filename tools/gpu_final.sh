# Final round call: gpu_round.sh, then the out-of-core runs with page-locked buffers
# (2048^3 and, when the box has the host memory, 4096 x 4096 x 2048).
cd $GRAFT_REPO_ROOT
TAG=${1:-final}
bash tools/gpu_round.sh $TAG
O=gpurun_out/$TAG
free -g > $O/free.txt 2>&1; cat $O/free.txt
AV=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
echo "MemAvailable GiB: $AV"
if [ "$AV" -gt 400 ]; then
timeout 900 python tools/bench_ooc.py --d 4096 --nz 2048 --pinned --reps 2 2>&1 | tail -1 > $O/ooc_4096x4096x2048_pinned.json; echo "ooc4096 rc=$?"
cut -c1-600 $O/ooc_4096x4096x2048_pinned.json
fi
