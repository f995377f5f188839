# interleaved A/B of library builds on one config: bash scripts/gpu_libab.sh <config> <reps> lib1 lib2 ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C=$1; R=$2; shift; shift
for r in $(seq 1 $R); do
  for L in "$@"; do
    ACA_LIB=$L timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/lab_$C_$L_$r.json 2>/dev/null
    python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['roofline']['mean_sweep_ms'],4))" gpurun_out/lab_$C_$L_$r.json "$C $L"
  done
done
