cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for VR in "3 2" "3 3" "3 4" "3 6" "0 3"; do set -- $VR
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rounds $2 --variant $1 > gpurun_out/bench_c3_V$1_R$2.log 2>&1; echo "bench V$1 R$2 rc=$?" >> gpurun_out/rc.txt
done
cat gpurun_out/rc.txt
