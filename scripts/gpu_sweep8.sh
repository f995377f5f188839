cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "early or class or variants" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for i in 1 2; do timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_rep$i.log 2>&1; echo "bench c3 rep$i rc=$?" >> gpurun_out/rc.txt; done
for BR in "1 3" "4 3" "32 3" "1 6" "4 6"; do set -- $BR
  ACA_BULK=$1 timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e --early-reject 1 --rounds $2 > gpurun_out/bench_c5_E1_B$1_R$2.log 2>&1; echo "bench c5 B$1 R$2 rc=$?" >> gpurun_out/rc.txt
done
cat gpurun_out/rc.txt
