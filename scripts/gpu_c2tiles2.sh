cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],2), round(d['roofline']['mean_sweep_ms'],4), d['roofline']['sweeps_per_step'])" $1 "$2"; }
for T in 64x64 32x32 64x32; do for R in 0 4 8 12; do
  timeout 300 python bench.py --config c2 --tile $T --rounds $R --steps 5 --no-cpu --no-e2e > gpurun_out/c2t_${T}_$R.json 2>/dev/null; line gpurun_out/c2t_${T}_$R.json "c2 $T R=$R"
done; done
ACA_TILE_NT=256 timeout 300 python bench.py --config c2 --steps 5 --no-cpu --no-e2e > gpurun_out/c2t_nt256.json 2>/dev/null; line gpurun_out/c2t_nt256.json "c2 64x64/256"
