# Quick parity + bench lines, then one ncu --set full capture (with source) of the tile kernel.
# usage: bash scripts/gpu_qprof.sh <tag>
cd $GRAFT_REPO_ROOT
TAG=${1:-qp}
bash scripts/gpu_quick.sh $TAG
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:tile_tma -s 40 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
