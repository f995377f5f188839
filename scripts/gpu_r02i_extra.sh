# r02i extras at HEAD: throughput of the q-th degree neighbourhood engine, and the race checks
# (repeated runs identical) re-run after the TMA L2-promotion change and the a10 write-back split.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/qnbr_bench.py > gpurun_out/qnbr_bench_r02i.jsonl 2> gpurun_out/qnbr_bench_r02i.err; echo "qnbr rc=$?"
cat gpurun_out/qnbr_bench_r02i.jsonl
R=scripts/repeat_check.py
{
python $R c5 15
python $R c5 15 class_book=0
python $R c5 20 "dims=(2048,2048)" max_ctas=7 T=60.0
python $R c3 20
python $R c4 20
python $R c2 30
} > gpurun_out/repeat_r02i.log 2>&1
echo "repeat rc=$?"; tail -12 gpurun_out/repeat_r02i.log
