cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for E in 0 1; do
  timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e --early-reject $E > gpurun_out/bench_c5_E$E.log 2>&1; echo "bench c5 E$E rc=$?" >> gpurun_out/rc.txt
done
for B in 1 4; do
  ACA_BULK=$B timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_B$B.log 2>&1; echo "bench c3 B$B rc=$?" >> gpurun_out/rc.txt
done
timeout 600 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt
