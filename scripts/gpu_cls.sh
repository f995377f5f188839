# a10 class bookkeeping: tests + c5 bench under several thresholds
# usage: bash scripts/gpu_cls.sh <tag>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-cls}
timeout 900 python -m pytest tests/test_gpu_classes.py tests/test_gpu_parity.py -m gpu -q -x -k "class or early" > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_$TAG.log
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --config c5"
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],1), d['firing_fraction'], d.get('a10'))" $1 "$2"; }
for W in -1 0.0005 0.002 0.01 1; do timeout 300 $B --early-reject 1 --class-book 1 --class-wmax $W > gpurun_out/cls_$W.json 2>gpurun_out/cls_$W.err; line gpurun_out/cls_$W.json "c5 wmax=$W"; done
timeout 300 $B --early-reject 0 > gpurun_out/cls_plain.json 2>/dev/null; line gpurun_out/cls_plain.json "c5 plain"
