# ncu evidence for the dominant kernel (run on one B200 via gpurun; see B200_PROFILING.md)
# usage: bash scripts/profile.sh <tag>
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --rounds ${ROUNDS:-3}"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/prof_plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_tma -s 20 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
