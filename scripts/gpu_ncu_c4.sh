# ncu --set full capture of the c4 (3-D) tile kernel + its launch list (r02h: 64 B TMA promotion)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${1:-r02h}
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_c4_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$TAG.csv $CMD > gpurun_out/ncu_launches_c4_$TAG.log 2>&1
echo "launches c4 rc=$?"
CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_grp -s 20 -c 1 -o /tmp/prof_c4_$TAG $CMD > gpurun_out/ncu_c4_$TAG.log 2>&1
echo "ncu c4 rc=$?"
ncu -i /tmp/prof_c4_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_c4_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_c4_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src_c4_$TAG.csv 2>/dev/null
gzip -f gpurun_out/ncu_src_c4_$TAG.csv
