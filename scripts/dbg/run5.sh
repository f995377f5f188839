cd $GRAFT_REPO_ROOT
ACA_SYNC_DEBUG=1 ACA_LIB=libaca_dbg.so timeout 300 python scripts/dbg/c5dbg4.py 8192x8192 1 2>&1 | tail -12
ACA_SYNC_DEBUG=1 timeout 300 python scripts/dbg/c5dbg4.py 8192x8192 1 2>&1 | tail -5
