cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
for M in 0 1 2; do for R in 3 4 6; do
  ACA_ROUND_MODE=$M timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rounds $R > gpurun_out/bench_c3_M${M}_R$R.log 2>&1; echo "bench M$M R$R rc=$?" >> gpurun_out/rc.txt
done; done
cat gpurun_out/rc.txt
