# work-list variant: parity + c3 sweep over R. usage: bash scripts/gpu_wl.sh <tag> [rounds...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-wl}; shift
RS=${@:-4 8 16 32}
rm -f gpurun_out/rc_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "variants or tiled or shard or compos or full" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_$TAG.txt
for R in $RS; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --variant 4 --rounds $R > gpurun_out/bench_${TAG}_V4_R$R.json 2>&1; echo "V4 R$R rc=$?" >> gpurun_out/rc_$TAG.txt
done
cat gpurun_out/rc_$TAG.txt
