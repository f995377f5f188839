# Jacobi (one launch over all tiles, checkerboard -1) vs checkerboard sweeps, per config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-jac}
for C in c3 c4 c5; do
  timeout 600 python bench.py --config $C --checkerboard -1 --steps 3 --no-cpu --no-e2e > gpurun_out/jac_${C}_$TAG.json 2> gpurun_out/jac_${C}_$TAG.err
  python scripts/bline.py gpurun_out/jac_${C}_$TAG.json "$C jacobi"
done
ACA_NO_RES=1 timeout 600 python bench.py --config c2 --steps 3 --no-cpu --no-e2e > gpurun_out/jac_c2cb_$TAG.json 2>&1; python scripts/bline.py gpurun_out/jac_c2cb_$TAG.json "c2 tile kernel checkerboard"
ACA_NO_RES=1 timeout 600 python bench.py --config c2 --checkerboard -1 --steps 3 --no-cpu --no-e2e > gpurun_out/jac_c2_$TAG.json 2>&1; python scripts/bline.py gpurun_out/jac_c2_$TAG.json "c2 tile kernel jacobi"
