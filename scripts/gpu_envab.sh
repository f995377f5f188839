# parity slice, then bench lines under env settings: bash scripts/gpu_envab.sh <tag> "<configs>" "ENV=a" "ENV=b" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1; CONFIGS=$2; shift; shift
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_classes.py -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_$TAG.log
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],1), round(d['roofline']['mean_sweep_ms'],3), d['roofline']['sweeps_per_step'], round(d['firing_fraction'],4))" $1 "$2"; }
i=0
for E in "$@"; do i=$((i+1))
  for C in $CONFIGS; do env $E timeout 300 python bench.py --config $C --steps 3 --no-cpu --no-e2e > gpurun_out/b_${TAG}_${i}_$C.json 2>/dev/null; line gpurun_out/b_${TAG}_${i}_$C.json "[$E] $C"; done
done
