# class bookkeeping (bit-sliced recount) check: class tests, c5 digests, c5 bench at several thresholds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-cls2}
timeout 900 python -m pytest tests/test_gpu_classes.py tests/test_gpu_fullsize.py -m gpu -q -x -k "class or c5" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for W in 0.01 -1 0.002 1; do
  timeout 600 python bench.py --config c5 --class-wmax $W --no-cpu --no-e2e > gpurun_out/c5_w${W}_$TAG.json 2> gpurun_out/c5_w${W}_$TAG.err
  python scripts/bline.py gpurun_out/c5_w${W}_$TAG.json "c5 wmax=$W"
done
timeout 600 python bench.py --config c5 --early-reject 0 --class-book 0 --no-cpu --no-e2e > gpurun_out/c5_plain_$TAG.json 2>&1
python scripts/bline.py gpurun_out/c5_plain_$TAG.json "c5 plain"
