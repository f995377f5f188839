# Round-2 quick iteration: GPU parity subset (-k expr), then bench lines of the given configs.
# usage: bash scripts/gpu_r2q.sh <tag> "<pytest -k expr>" "c3 c4 c5 c2"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-q}
K=${2:-"not fullsize"}
CONFS=${3:-"c3"}
timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pq_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pq_$TAG.log
for C in $CONFS; do
  timeout 600 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/bq_${C}_$TAG.json 2> gpurun_out/bq_${C}_$TAG.err
  python -c "
import json; d=json.loads(open('gpurun_out/bq_${C}_$TAG.json').read().strip().splitlines()[-1]); print('$C', '%.4e'%d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('config',{}).get('sweeps'))" || tail -3 gpurun_out/bq_${C}_$TAG.err
done
