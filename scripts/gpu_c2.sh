# c2 bench over R and checkerboard on/off
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for CB in 0 -1; do for R in 8 16; do
  timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --rounds $R --checkerboard $CB > gpurun_out/bench_c2cb_${CB}_R$R.json 2>&1; echo "CB$CB R$R rc=$?"
done; done
