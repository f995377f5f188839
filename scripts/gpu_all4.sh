# quick: a pytest subset ($2) then c3, c4, c5 (default + a10 only) bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-all4}
if [ -n "$2" ]; then timeout 1200 python -m pytest $2 -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log; fi
for C in c3 c4 c5 c2; do
  timeout 300 python bench.py --config $C --steps 3 --no-cpu --no-e2e > gpurun_out/q_${C}_$TAG.json 2> gpurun_out/q_${C}_$TAG.err; python scripts/bline.py gpurun_out/q_${C}_$TAG.json "$C"
done
timeout 300 python bench.py --config c5 --class-book 0 --steps 3 --no-cpu --no-e2e > gpurun_out/q_c5a10_$TAG.json 2>&1; python scripts/bline.py gpurun_out/q_c5a10_$TAG.json "c5 a10 only"
