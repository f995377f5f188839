cd $GRAFT_REPO_ROOT
bash scripts/gpu_quick.sh pm9
for T in 64x128; do for R in 5 6 8; do
  timeout 600 python bench.py --config c3 --no-cpu --no-e2e --tile $T --rounds $R > gpurun_out/bt_${T}_R$R.json 2>gpurun_out/bt_${T}_R$R.err
  python scripts/bline.py gpurun_out/bt_${T}_R$R.json ${T}_R$R
done; done
