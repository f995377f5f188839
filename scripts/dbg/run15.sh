cd $GRAFT_REPO_ROOT
H='{"phys": {"beta": 0.4406868, "h": 0.0, "rule": 0, "init_q": 0.5}, "T": 20.0}'
P="timeout 100 python scripts/dbg/c5dbg5.py 8192x8192"
$P "$H"; $P '{"rounds_per_launch": 8}'; $P '{}'; $P '{"checkerboard": -1}'
timeout 200 python scripts/dbg/c5dbg4.py 8192x8192 1 2>&1 | tail -3
bash scripts/gpu_r2q.sh a2 "not fullsize and not bench_multiproc and not onsager" "c3 c4 c5 c2"
