# full GPU suite + c3/c4/c5 bench lines (no cpu/e2e legs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-pipe}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pt_$TAG.log
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],1), d['roofline']['frac'], d['roofline']['survey_8d']['frac'])" $1 "$2"; }
for C in c3 c4 c5 c2; do timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/b_${C}_$TAG.json 2>gpurun_out/b_${C}_$TAG.err; line gpurun_out/b_${C}_$TAG.json $C; done
timeout 300 python bench.py --config c5 --early-reject 0 --class-book 0 --no-cpu --no-e2e > gpurun_out/b_c5p_$TAG.json 2>/dev/null; line gpurun_out/b_c5p_$TAG.json c5plain
