set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for V in 0 3; do for R in 2 3 4; do
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rounds $R --variant $V > gpurun_out/bench_c3_V${V}_R$R.log 2>&1; echo "bench V$V R$R rc=$?" >> gpurun_out/rc.txt
done; done
cat gpurun_out/rc.txt
