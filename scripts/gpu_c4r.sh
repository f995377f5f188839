# c4 in-tile rounds 4 vs 5, interleaved A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-c4r}
for i in 1 2; do for R in 4 5; do
  timeout 600 python bench.py --config c4 --rounds $R --no-cpu --no-e2e > gpurun_out/c4r${R}_${i}_$TAG.json 2>/dev/null; python scripts/bline.py gpurun_out/c4r${R}_${i}_$TAG.json "c4 R=$R run $i"
done; done
