# quick c5 lines: class + a10 (default), a10 only, plain; optional pytest subset as $2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-c5q}
if [ -n "$2" ]; then timeout 1200 python -m pytest $2 -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log; fi
timeout 600 python bench.py --config c5 --steps 3 --no-cpu --no-e2e > gpurun_out/c5_def_$TAG.json 2> gpurun_out/c5_def_$TAG.err; python scripts/bline.py gpurun_out/c5_def_$TAG.json "c5 default"
timeout 600 python bench.py --config c5 --class-book 0 --steps 3 --no-cpu --no-e2e > gpurun_out/c5_a10_$TAG.json 2>&1; python scripts/bline.py gpurun_out/c5_a10_$TAG.json "c5 a10 only"
timeout 600 python bench.py --config c5 --early-reject 0 --class-book 0 --steps 3 --no-cpu --no-e2e > gpurun_out/c5_plain_$TAG.json 2>&1; python scripts/bline.py gpurun_out/c5_plain_$TAG.json "c5 plain"
