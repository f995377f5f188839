# a10 fast fire check: every test that runs the a10 path, then c5 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-a10}
timeout 1200 python -m pytest $(grep -l "early_reject" tests/test_gpu*.py) -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for W in 0.01 1 -1 0.05; do
  timeout 600 python bench.py --config c5 --class-wmax $W --no-cpu --no-e2e > gpurun_out/c5_w${W}_$TAG.json 2> gpurun_out/c5_w${W}_$TAG.err
  python scripts/bline.py gpurun_out/c5_w${W}_$TAG.json "c5 wmax=$W"
done
timeout 600 python bench.py --config c5 --class-book 0 --no-cpu --no-e2e > gpurun_out/c5_a10only_$TAG.json 2>&1
python scripts/bline.py gpurun_out/c5_a10only_$TAG.json "c5 a10 no class"
