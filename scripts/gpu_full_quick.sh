# Full GPU test suite + c3/c2/c5 bench lines. usage: bash scripts/gpu_full_quick.sh <tag>
cd $GRAFT_REPO_ROOT
TAG=${1:-fq}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
for C in c3 c2 c4 c5; do
  timeout 600 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/bq_${C}_$TAG.json 2> gpurun_out/bq_${C}_$TAG.err
  python scripts/bline.py gpurun_out/bq_${C}_$TAG.json $C
done
