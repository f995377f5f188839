# c4 (3-D) bench over variant x R: usage bash scripts/gpu_c4.sh "<variants>" "<rounds>"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for V in $1; do for R in $2; do
  timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e --variant $V --rounds $R > gpurun_out/bench_c4v_V${V}_R$R.json 2>&1; echo "V$V R$R rc=$?"
done; done
