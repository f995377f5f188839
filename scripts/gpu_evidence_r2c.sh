# Round-2 (r02c) evidence: bench lines of every config (e2e + cpu baseline), c5 plain path, the reference
# arm, virtual shard + per-GPU strip runs, ncu launch list of the default bench, and full captures
# (with source pages) of each config's tile kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02c}
RC=gpurun_out/rc_$TAG.txt; rm -f $RC
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> $RC
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?" >> $RC
for C in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $C > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; echo "bench $C rc=$?" >> $RC
done
timeout 900 python bench.py --config c5 --early-reject 0 --class-book 0 > gpurun_out/bench_c5plain_$TAG.json 2> gpurun_out/bench_c5plain_$TAG.err; echo "bench c5plain rc=$?" >> $RC
for G in 2 4 8; do
  timeout 600 python bench.py --shards $G --no-cpu --no-e2e > gpurun_out/bench_c3_g${G}_$TAG.json 2>> gpurun_out/shards_$TAG.err
  timeout 600 python bench.py --config c4 --shards $G --no-cpu --no-e2e > gpurun_out/bench_c4_g${G}_$TAG.json 2>> gpurun_out/shards_$TAG.err
  timeout 600 python bench.py --rows-div $G --no-cpu --no-e2e > gpurun_out/bench_c3_rd${G}_$TAG.json 2>> gpurun_out/shards_$TAG.err
  timeout 600 python bench.py --config c4 --rows-div $G --no-cpu --no-e2e > gpurun_out/bench_c4_rd${G}_$TAG.json 2>> gpurun_out/shards_$TAG.err
done
echo "shards done" >> $RC
nproc > gpurun_out/host_$TAG.txt; lscpu | head -20 >> gpurun_out/host_$TAG.txt; nvidia-smi >> gpurun_out/host_$TAG.txt
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?" >> $RC
for C in ${NCU_CONFIGS:-c3 c4 c5 c2}; do
  CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_grp -s 20 -c 1 -o /tmp/prof_${C}_$TAG $CMD > gpurun_out/ncu_${C}_$TAG.log 2>&1
  echo "ncu $C rc=$?" >> $RC
  ncu -i /tmp/prof_${C}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${C}_$TAG.csv 2>/dev/null
  ncu -i /tmp/prof_${C}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src_${C}_$TAG.csv 2>/dev/null
  gzip -f gpurun_out/ncu_src_${C}_$TAG.csv
done
cat $RC
