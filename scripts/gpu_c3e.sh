# c3 / c4 / c2 with the a10 early rejection (exact; the same trajectory) vs plain
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-c3e}
for i in 1 2; do
timeout 600 python bench.py --config c3 --early-reject 1 --steps 3 --no-cpu --no-e2e > gpurun_out/c3e_${i}_$TAG.json 2>gpurun_out/c3e_${i}_$TAG.err; python scripts/bline.py gpurun_out/c3e_${i}_$TAG.json "c3 a10"
timeout 600 python bench.py --config c3 --steps 3 --no-cpu --no-e2e > gpurun_out/c3p_${i}_$TAG.json 2>/dev/null; python scripts/bline.py gpurun_out/c3p_${i}_$TAG.json "c3 plain"
done
timeout 600 python bench.py --config c4 --early-reject 1 --steps 3 --no-cpu --no-e2e > gpurun_out/c4e_$TAG.json 2>gpurun_out/c4e_$TAG.err; python scripts/bline.py gpurun_out/c4e_$TAG.json "c4 a10"
timeout 600 python bench.py --config c2 --early-reject 1 --steps 3 --no-cpu --no-e2e > gpurun_out/c2e_$TAG.json 2>gpurun_out/c2e_$TAG.err; python scripts/bline.py gpurun_out/c2e_$TAG.json "c2 a10 (tile kernel)"
