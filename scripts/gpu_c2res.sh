cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_res.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_res.log
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],3), d['roofline']['sweeps_per_step'])" $1 "$2"; }
for R in 3 4 5 6 8 10 12 16; do timeout 300 python bench.py --config c2 --rounds $R --steps 10 --no-cpu --no-e2e > gpurun_out/c2res_$R.json 2>/dev/null; line gpurun_out/c2res_$R.json "c2 res R=$R"; done
