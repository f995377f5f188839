cd $GRAFT_REPO_ROOT
run() { env $2 timeout 600 python bench.py --config c2 --no-cpu --no-e2e $3 > gpurun_out/bc2_$1.json 2>/dev/null; python scripts/bline.py gpurun_out/bc2_$1.json $1; }
run 64x64_R6 "X=1" "--rounds 6"
run 32x32_R6 "X=1" "--tile 32x32 --rounds 6"
run 32x32_R10 "X=1" "--tile 32x32 --rounds 10"
run 64x32nt128_R6 "ACA_TILE_NT=128" "--tile 64x32 --rounds 6"
run 64x32nt128_R8 "ACA_TILE_NT=128" "--tile 64x32 --rounds 8"
run 64x32nt256_R8 "ACA_TILE_NT=256" "--tile 64x32 --rounds 8"
