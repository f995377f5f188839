# a10 ablation: c5 / c3 with early rejection on and off, bulk settings; per-GPU strip workloads
# usage: bash scripts/gpu_early.sh <tag>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-e}
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('firing_fraction'))" $1 "$2"; }
for E in 1 0; do timeout 300 $B --config c5 --early-reject $E > gpurun_out/e_c5_$E.json 2>/dev/null; line gpurun_out/e_c5_$E.json "c5 early=$E"; done
for BU in 4; do ACA_BULK=$BU timeout 300 $B --config c5 > gpurun_out/e_c5_b$BU.json 2>/dev/null; line gpurun_out/e_c5_b$BU.json "c5 bulk=$BU"; done
timeout 300 $B --config c3 --early-reject 1 > gpurun_out/e_c3_1.json 2>/dev/null; line gpurun_out/e_c3_1.json "c3 early=1"
for G in 2 4 8; do timeout 300 $B --rows-div $G > gpurun_out/rd_c3_$G.json 2>/dev/null; line gpurun_out/rd_c3_$G.json "c3 rows-div=$G";
  timeout 300 $B --config c4 --rows-div $G > gpurun_out/rd_c4_$G.json 2>/dev/null; line gpurun_out/rd_c4_$G.json "c4 rows-div=$G"; done
