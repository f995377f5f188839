cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for X in 32x16x8:4 32x16x8:6 16x16x16:4 16x16x16:6 32x32x8:4 8x8x8:4; do T=${X%%:*}; R=${X##*:}
  timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e --tile $T --rounds $R > gpurun_out/bench_c4s_${T}_R$R.json 2>&1; echo "$X rc=$?"
done
