# c5 class-on-plain overhead ablations (variant libraries built by scripts/build_var.sh)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-clsab}
for L in libaca.so libaca_nocount.so libaca_noarm.so libaca_nocountarm.so; do
  ACA_LIB=$L timeout 600 python bench.py --config c5 --class-wmax -1 --steps 3 --no-cpu --no-e2e > gpurun_out/c5ab_${L}_$TAG.json 2> gpurun_out/c5ab_${L}_$TAG.err
  python scripts/bline.py gpurun_out/c5ab_${L}_$TAG.json "c5 wmax=-1 $L"
done
timeout 600 python bench.py --config c5 --early-reject 0 --class-book 0 --steps 3 --no-cpu --no-e2e > gpurun_out/c5ab_plain_$TAG.json 2>&1
python scripts/bline.py gpurun_out/c5ab_plain_$TAG.json "c5 plain"
