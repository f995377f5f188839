cd $GRAFT_REPO_ROOT
export ACA_SYNC_DEBUG=1 ACA_LIB=libaca_dbg.so
H='{"phys": {"beta": 0.4406868, "h": 0.0, "rule": 0, "init_q": 0.5}, "T": 20.0}'
timeout 300 python scripts/dbg/c5dbg5.py 8192x8192 "$H"
timeout 300 python scripts/dbg/c5dbg5.py 8192x8192 '{"rounds_per_launch": 8}'
