# c3 bench under env settings: usage: bash scripts/gpu_env.sh <tag> "<bench args>" "ENV=a ENV2=b" "ENV=c" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1; ARGS=$2; shift; shift
i=0
for E in "$@"; do i=$((i+1))
  env $E timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e $ARGS > gpurun_out/bench_${TAG}_$i.json 2>&1; echo "$i [$E] rc=$?"
done
