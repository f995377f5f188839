# EM=2 (class bookkeeping) overhead on the a10 path: one tile_rounds instance, no count / arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-clsab2}
for L in libaca.so libaca_eo.so libaca_eo_nc.so; do
  ACA_LIB=$L timeout 600 python bench.py --config c5 --class-wmax 1 --steps 3 --no-cpu --no-e2e > gpurun_out/c5ab_${L}_$TAG.json 2> gpurun_out/c5ab_${L}_$TAG.err
  python scripts/bline.py gpurun_out/c5ab_${L}_$TAG.json "c5 wmax=1 $L"
done
timeout 600 python bench.py --config c5 --class-book 0 --steps 3 --no-cpu --no-e2e > gpurun_out/c5ab_a10_$TAG.json 2>&1
python scripts/bline.py gpurun_out/c5ab_a10_$TAG.json "c5 a10 no class"
