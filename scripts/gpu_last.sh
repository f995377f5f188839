# last check of the round: full GPU suite, smoke, default bench line, c4 line (new traffic figure)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_last.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_last.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_last.log
timeout 900 python bench.py > gpurun_out/bench_last.json 2> gpurun_out/bench_last.err; echo "bench rc=$?"; cat gpurun_out/bench_last.json
timeout 900 python bench.py --config c4 --no-cpu > gpurun_out/bench_c4_last.json 2> gpurun_out/bench_c4_last.err; echo "bench c4 rc=$?"
