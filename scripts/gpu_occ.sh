# occupancy check: parity + c3 R4/R6 + c4 + c5 bench lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_occ.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_occ.log
for R in 4 6; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --rounds $R > gpurun_out/bench_occ_c3_R$R.json 2>&1; done
timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_occ_c4.json 2>&1
timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_occ_c5.json 2>&1
echo done
