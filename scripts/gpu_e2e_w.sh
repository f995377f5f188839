# e2e leg with its own untimed warm-up: default bench twice, c2, c4, c5 (device value next to e2e)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for C in c3 c3 c2 c2 c4 c5 c1; do
  timeout 900 python bench.py --config $C --no-cpu > gpurun_out/e2ew_$C.json 2> gpurun_out/e2ew_$C.err; echo "$C rc=$?"
  python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], '%.4e'%d['e2e']['value'], round(d['e2e']['value']/d['value'],3))" gpurun_out/e2ew_$C.json $C
done
timeout 600 python -m pytest tests -m gpu -q -x -k "bench or ipc" 2>&1 | tail -3
