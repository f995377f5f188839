# interleaved A/B of library builds: bench lines of c3/c4/c5 (x2), parity slice on the last build
# usage: bash scripts/gpu_ab2.sh <tag> "<libA> <libB>"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab2}; LIBS=${2:-libaca.so}
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],2), round(d['roofline']['mean_sweep_ms'],4), d['roofline']['sweeps_per_step'])" $1 "$2"; }
for rep in 1 2; do for C in ${CONFIGS:-c3 c4 c5}; do for L in $LIBS; do
  ACA_LIB=$L timeout 300 python bench.py --config $C --steps 5 --no-cpu --no-e2e > gpurun_out/${TAG}_${L}_${C}_$rep.json 2>/dev/null; line gpurun_out/${TAG}_${L}_${C}_$rep.json "$L $C rep=$rep"
done; done; done
for L in $LIBS; do LAST=$L; done
ACA_LIB=$LAST timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_classes.py tests/test_gpu_frames.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "$LAST pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
