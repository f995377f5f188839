cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for DR in "0 3" "1 3" "1 4" "1 6"; do set -- $DR
  ACA_DEFER=$1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --rounds $2 > gpurun_out/bench_c3_D$1_R$2.log 2>&1; echo "bench D$1 R$2 rc=$?" >> gpurun_out/rc.txt
done
cat gpurun_out/rc.txt
