# Quick iteration: parity of the tiled paths + c3/c2 bench lines (no ncu).
# usage: bash scripts/gpu_quick.sh <tag> [extra pytest -k expr]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-q}
K=${2:-"tiled or variant or fullsize or shard or law or life or early or frames"}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_frames.py -m gpu -q -x -k "$K" > gpurun_out/pq_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pq_$TAG.log
for C in c3 c2 c5; do
  timeout 600 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/bq_${C}_$TAG.json 2> gpurun_out/bq_${C}_$TAG.err
  python -c "
import json; d=json.loads(open('gpurun_out/bq_${C}_$TAG.json').read().strip().splitlines()[-1]); print('$C', '%.4e'%d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
