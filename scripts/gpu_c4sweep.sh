cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],2), round(d['roofline']['mean_sweep_ms'],4), d['roofline']['sweeps_per_step'])" $1 "$2"; }
for T in 32x16x8 16x16x16; do for R in 3 4 5 6 8; do
  timeout 300 python bench.py --config c4 --tile $T --rounds $R --steps 3 --no-cpu --no-e2e > gpurun_out/c4t_${T}_$R.json 2>/dev/null; line gpurun_out/c4t_${T}_$R.json "c4 $T R=$R"
done; done
for R in 4 6 7; do timeout 300 python bench.py --config c3 --rounds $R --steps 3 --no-cpu --no-e2e > gpurun_out/c3r_$R.json 2>/dev/null; line gpurun_out/c3r_$R.json "c3 R=$R"; done
