# r02c: GPU suite slice for the latest changes, bench c3/c5 lines, ncu full capture of c3's tile kernel (source pages)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_classes.py -m gpu -q -x > gpurun_out/pt_r2c.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_r2c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2c.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2c.log
for C in c5; do timeout 600 python bench.py --config $C > gpurun_out/bench_${C}_r2c.json 2> gpurun_out/bench_${C}_r2c.err; echo "bench $C rc=$?"; done
timeout 600 python bench.py --config c5 --early-reject 0 --class-book 0 --no-cpu > gpurun_out/bench_c5plain_r2c.json 2>/dev/null
C=c3; CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_grp -s 30 -c 1 -o /tmp/prof_${C}_r2c $CMD > gpurun_out/ncu_${C}_r2c.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_${C}_r2c.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${C}_r2c.csv 2>/dev/null
ncu -i /tmp/prof_${C}_r2c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src_${C}_r2c.csv 2>/dev/null
gzip -f gpurun_out/ncu_src_${C}_r2c.csv
