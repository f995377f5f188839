# parity + c3 sweep over "variant:tile:rounds" triples. usage: bash scripts/gpu_tiles.sh <tag> 0:64x64:4 ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1; shift
rm -f gpurun_out/rc_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_$TAG.txt
for X in "$@"; do V=$(echo $X | cut -d: -f1); T=$(echo $X | cut -d: -f2); R=$(echo $X | cut -d: -f3)
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --variant $V --tile $T --rounds $R > gpurun_out/bench_${TAG}_V${V}_${T}_R$R.json 2>&1; echo "$X rc=$?" >> gpurun_out/rc_$TAG.txt
done
cat gpurun_out/rc_$TAG.txt
