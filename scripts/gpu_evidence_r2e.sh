# Round-2 (r02e) evidence: full GPU suite, smoke, bench lines of every config (e2e + cpu baseline),
# c5 a10-only and plain lines, the reference arm, the launch list of the default bench, and full
# ncu captures (with source pages) of the c3 and c5 tile kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02e}
RC=gpurun_out/rc_$TAG.txt; rm -f $RC
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $RC; tail -3 gpurun_out/pytest_gpu_$TAG.log >> $RC
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $RC
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> $RC
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?" >> $RC
for C in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $C > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; echo "bench $C rc=$?" >> $RC
done
timeout 900 python bench.py --config c5 --class-book 0 > gpurun_out/bench_c5a10_$TAG.json 2> gpurun_out/bench_c5a10_$TAG.err; echo "bench c5a10 rc=$?" >> $RC
timeout 900 python bench.py --config c5 --early-reject 0 --class-book 0 > gpurun_out/bench_c5plain_$TAG.json 2> gpurun_out/bench_c5plain_$TAG.err; echo "bench c5plain rc=$?" >> $RC
nproc > gpurun_out/host_$TAG.txt; lscpu | head -20 >> gpurun_out/host_$TAG.txt; nvidia-smi >> gpurun_out/host_$TAG.txt
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?" >> $RC
CMD="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_c5_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$TAG.csv $CMD > gpurun_out/ncu_launches_c5_$TAG.log 2>&1
echo "launches c5 rc=$?" >> $RC
for C in ${NCU_CONFIGS:-c5 c3}; do
  CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_grp -s 20 -c 1 -o /tmp/prof_${C}_$TAG $CMD > gpurun_out/ncu_${C}_$TAG.log 2>&1
  echo "ncu $C rc=$?" >> $RC
  ncu -i /tmp/prof_${C}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${C}_$TAG.csv 2>/dev/null
  ncu -i /tmp/prof_${C}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src_${C}_$TAG.csv 2>/dev/null
  gzip -f gpurun_out/ncu_src_${C}_$TAG.csv
done
cat $RC
