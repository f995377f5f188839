set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for R in 2 4 8 16 64; do
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rounds $R > gpurun_out/bench_c3_R$R.log 2>&1; echo "bench R$R rc=$?" >> gpurun_out/rc.txt
done
cat gpurun_out/rc.txt
