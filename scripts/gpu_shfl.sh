# A/B of the left/right high halves by warp shuffle (libaca_shfl.so, -DACA_SHFL_LR) against the
# 32-bit shared loads (default), interleaved; then the parity tests of the 2-D tile paths on the variant.
# build the variant first (here, before gpurun): bash scripts/build_var.sh libaca_shfl.so -DACA_SHFL_LR
cd $GRAFT_REPO_ROOT
bash scripts/gpu_libab.sh c3 3 libaca.so libaca_shfl.so
bash scripts/gpu_libab.sh c2 2 libaca.so libaca_shfl.so
ACA_LIB=libaca_shfl.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties_nbcap.py -m gpu -q -x 2>&1 | tail -3
