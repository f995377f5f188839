# full ncu capture (with source) of the c5 a10-only kernel (EM=1), to compare with the class kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-em1}
CMD="python bench.py --config c5 --class-book 0 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_grp -s 20 -c 1 -o /tmp/prof_em1 $CMD > gpurun_out/ncu_em1_$TAG.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_em1.ncu-rep --page raw --csv > gpurun_out/ncu_raw_em1_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_em1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src_em1_$TAG.csv 2>/dev/null
gzip -f gpurun_out/ncu_src_em1_$TAG.csv
CMD="python bench.py --config c5 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_grp -s 20 -c 1 -o /tmp/prof_em2 $CMD > gpurun_out/ncu_em2_$TAG.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_em2.ncu-rep --page raw --csv > gpurun_out/ncu_raw_em2_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_em2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src_em2_$TAG.csv 2>/dev/null
gzip -f gpurun_out/ncu_src_em2_$TAG.csv
