cd $GRAFT_REPO_ROOT
export ACA_SYNC_DEBUG=1 ACA_LIB=libaca_dbg.so
P="timeout 120 python scripts/dbg/c5dbg5.py"
$P 8192x8192 '{"phys": {"beta": 0.4406868, "h": 0.0, "rule": 0, "init_q": 0.5}, "T": 20.0}'
$P 8192x8192 '{}'
