# quick check: GPU tests + c3 bench (+ optional extra bench args)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_q$i.log 2>&1; echo "bench c3 q$i rc=$?" >> gpurun_out/rc.txt; done
timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5_q.log 2>&1; echo "bench c5 rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt
