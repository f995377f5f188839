# ncu full capture (source-attributed) of the tile kernel for the given configs.
# usage: bash scripts/gpu_prof_r2.sh <tag> "c3 c4"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-p}
for C in ${2:-c3}; do
  CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e"
  $CMD > gpurun_out/prof_plain_${C}_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_grp -s 30 -c 1 -o gpurun_out/prof_${C}_$TAG $CMD > gpurun_out/ncu_${C}_$TAG.log 2>&1
  echo "$C ncu rc=$?"
done
