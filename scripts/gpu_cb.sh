# checkerboard sweeps: parity + c3 sweep over variant x R. usage: bash scripts/gpu_cb.sh <tag> "<variants>" "<rounds>"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-cb}; VS=${2:-0 4}; RS=${3:-3 4 6 8}
rm -f gpurun_out/rc_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_$TAG.txt
for V in $VS; do for R in $RS; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --variant $V --rounds $R > gpurun_out/bench_${TAG}_V${V}_R$R.json 2>&1; echo "V$V R$R rc=$?" >> gpurun_out/rc_$TAG.txt
done; done
cat gpurun_out/rc_$TAG.txt
