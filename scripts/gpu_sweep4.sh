set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for VR in "0 2" "0 3" "0 4" "2 3" "1 3"; do set -- $VR
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rounds $2 --variant $1 > gpurun_out/bench_c3_V$1_R$2.log 2>&1; echo "bench V$1 R$2 rc=$?" >> gpurun_out/rc.txt
done
cat gpurun_out/rc.txt
