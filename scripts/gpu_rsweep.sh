# bench over in-tile rounds per visit R. usage: CFG=c3 bash scripts/gpu_rsweep.sh <tag> "3 4 5 6"
cd $GRAFT_REPO_ROOT
TAG=${1:-rs}
for R in ${2:-3 4 5 6}; do
  timeout 600 python bench.py --config ${CFG:-c3} --no-cpu --no-e2e --rounds $R > gpurun_out/br_${TAG}_R$R.json 2>/dev/null
  python scripts/bline.py gpurun_out/br_${TAG}_R$R.json R$R
done
