# c2 bench over R (and checkerboard on/off via ACA env not available: variant only)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for R in 4 8 16 32 64; do
  timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --rounds $R > gpurun_out/bench_c2r_R$R.json 2>&1; echo "R$R rc=$?"
done
