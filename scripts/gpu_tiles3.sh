# c4 over 3-D tile shapes. usage: bash scripts/gpu_tiles3.sh
cd $GRAFT_REPO_ROOT
run() {  # label, args
  timeout 600 python bench.py --config c4 --no-cpu --no-e2e $2 > gpurun_out/bt3_$1.json 2>gpurun_out/bt3_$1.err
  python scripts/bline.py gpurun_out/bt3_$1.json $1
}
run 32x16x8_R5 "--tile 32x16x8 --rounds 5"
run 16x16x16_R5 "--tile 16x16x16 --rounds 5"
run 16x16x16_R8 "--tile 16x16x16 --rounds 8"
run 32x32x8_R5 "--tile 32x32x8 --rounds 5"
run 32x32x8_R8 "--tile 32x32x8 --rounds 8"
