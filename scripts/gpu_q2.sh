cd $GRAFT_REPO_ROOT
bash scripts/gpu_quick.sh pm2
for D in 0 1; do
  ACA_DEFER_TAIL=$D timeout 600 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/bq_dt$D.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bq_dt$D.json').read().strip().splitlines()[-1]); print('dt$D', '%.4e'%d['value'], d['ms_per_step'], d['arrivals_per_cell_per_sweep'], d['roofline']['sweeps_per_step'], d['roofline']['mean_sweep_ms'])"
done
