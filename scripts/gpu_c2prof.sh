cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2_res.json 2>/dev/null; tail -c 400 gpurun_out/bench_c2_res.json
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:res_kernel -s 2 -c 1 -o /tmp/prof_c2res $CMD > gpurun_out/ncu_c2res.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_c2res.ncu-rep --page raw --csv > gpurun_out/ncu_raw_c2res.csv 2>/dev/null
ncu -i /tmp/prof_c2res.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src_c2res.csv 2>/dev/null; gzip -f gpurun_out/ncu_src_c2res.csv
