cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for L in libaca.so libaca_old.so libaca.so; do echo "== $L"; ACA_LIB=$L timeout 300 python scripts/e2e_diag.py c5 2>&1 | tail -12; done > gpurun_out/e2e_diag.txt
for L in libaca.so libaca_old.so; do ACA_LIB=$L timeout 300 python bench.py --config c5 --steps 5 --no-cpu > gpurun_out/e2e_b_$L.json 2>&1; done
cat gpurun_out/e2e_diag.txt
