set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt
