# 3-D parity subset + c4 bench. usage: bash scripts/gpu_c4q.sh <tag>
cd $GRAFT_REPO_ROOT
TAG=${1:-c4q}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_frames.py tests/test_gpu_ipc.py -m gpu -q -x > gpurun_out/pq3_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pq3_$TAG.log
for R in 5 6; do
timeout 600 python bench.py --config c4 --no-cpu --no-e2e --rounds $R > gpurun_out/bq_c4_${TAG}_R$R.json 2> gpurun_out/bq_c4_$TAG.err
python scripts/bline.py gpurun_out/bq_c4_${TAG}_R$R.json c4_R$R
done
