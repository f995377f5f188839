cd $GRAFT_REPO_ROOT
export ACA_SYNC_DEBUG=1
P="timeout 120 python scripts/dbg/c5dbg5.py"
$P 8192x8192 '{}'
$P 8192x8192 '{"checkerboard": -1}'
$P 8192x8192 '{"rounds_per_launch": 1}'
$P 8192x8192 '{"rounds_per_launch": 8}'
$P 8192x8192 '{"max_ctas": 16}'
$P 8192x8192 '{"event_hash": 0}'
$P 8192x8192 '{"phys": {"beta": 0.4406868, "h": 0.0, "rule": 0, "init_q": 0.5}, "T": 20.0}'
$P 8192x4096 '{}'
$P 6144x6144 '{}'
$P 8192x8192 '{"T": 100.0}'
$P 8192x8192 '{"early_reject": 0}'
