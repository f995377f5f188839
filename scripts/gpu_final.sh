# Round-end style evidence: full GPU tests, smoke, default bench line, reference arm, the other
# configs' bench lines, ncu launch list + full capture of the dominant kernel.
# usage: bash scripts/gpu_final.sh <tag>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
rm -f gpurun_out/rc_$TAG.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/rc_$TAG.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "bench ref rc=$?" >> gpurun_out/rc_$TAG.txt
for C in c2 c4 c5; do
  timeout 900 python bench.py --config $C --no-cpu > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; echo "bench $C rc=$?" >> gpurun_out/rc_$TAG.txt
done
nproc > gpurun_out/host_$TAG.txt; lscpu | head -20 >> gpurun_out/host_$TAG.txt
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?" >> gpurun_out/rc_$TAG.txt
$CMD > gpurun_out/prof_plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_tma -s 40 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?" >> gpurun_out/rc_$TAG.txt
cat gpurun_out/rc_$TAG.txt
