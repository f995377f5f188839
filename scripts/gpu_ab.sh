# A/B of library builds: parity slice + c3/c4/c5 bench lines per build (ACA_LIB) and env
# usage: bash scripts/gpu_ab.sh <tag> "<lib1> <lib2> ..."
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab}
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],1), round(d['roofline']['mean_sweep_ms'],3), d['roofline']['sweeps_per_step'])" $1 "$2"; }
for L in ${2:-libaca.so}; do
  ACA_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_classes.py -m gpu -q -x > gpurun_out/pt_${TAG}_$L.log 2>&1; echo "$L pytest rc=$?"; tail -2 gpurun_out/pt_${TAG}_$L.log
  for C in c3 c4 c5; do ACA_LIB=$L timeout 300 python bench.py --config $C --steps 3 --no-cpu --no-e2e > gpurun_out/b_${TAG}_${L}_$C.json 2>/dev/null; line gpurun_out/b_${TAG}_${L}_$C.json "$L $C"; done
  ACA_NO_TMA_BOX=1 ACA_LIB=$L timeout 300 python bench.py --config c3 --steps 3 --no-cpu --no-e2e > gpurun_out/b_${TAG}_${L}_c3nobox.json 2>/dev/null; line gpurun_out/b_${TAG}_${L}_c3nobox.json "$L c3 nobox"
done
