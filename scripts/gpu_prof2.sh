# bench + ncu full capture of one tile-kernel launch for each "variant:rounds" arg. usage: bash scripts/gpu_prof2.sh <tag> 0:4 4:6 ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1; shift
for VR in "$@"; do V=${VR%%:*}; R=${VR##*:}
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --variant $V --rounds $R"
  timeout 300 $CMD > gpurun_out/bench_${TAG}_V${V}_R$R.json 2>&1; echo "bench V$V R$R rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_tma -s 40 -c 1 -o gpurun_out/prof_${TAG}_V${V}_R$R $CMD > gpurun_out/ncu_${TAG}_V${V}_R$R.log 2>&1; echo "ncu V$V R$R rc=$?"
done
