cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "nccl" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for TV in "64x64 0" "64x64 2" "64x32 0" "64x32 2" "128x64 0" "32x32 0"; do set -- $TV
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --tile $1 --variant $2 > gpurun_out/bench_c3_T$1_V$2.log 2>&1; echo "bench T$1 V$2 rc=$?" >> gpurun_out/rc.txt
done
cat gpurun_out/rc.txt
