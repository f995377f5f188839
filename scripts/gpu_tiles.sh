# c3 over tile shapes / block sizes. usage: bash scripts/gpu_tiles.sh
cd $GRAFT_REPO_ROOT
run() {  # label, env, args
  env $2 timeout 600 python bench.py --config c3 --no-cpu --no-e2e $3 > gpurun_out/bt_$1.json 2>gpurun_out/bt_$1.err
  python scripts/bline.py gpurun_out/bt_$1.json $1
}
run 64x32_nt256_R5 "ACA_TILE_NT=256" "--tile 64x32 --rounds 5"
run 64x32_nt128_R5 "ACA_TILE_NT=128" "--tile 64x32 --rounds 5"
run 64x32_nt128_R6 "ACA_TILE_NT=128" "--tile 64x32 --rounds 6"
run 64x32_nt128_R4 "ACA_TILE_NT=128" "--tile 64x32 --rounds 4"
run 64x64_R5 "X=1" ""
