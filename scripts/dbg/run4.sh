cd $GRAFT_REPO_ROOT
ACA_LIB=libaca_dbg.so timeout 200 python scripts/dbg/c5dbg4.py 8192x8192 1 2>&1 | tail -12
timeout 200 python scripts/dbg/c5dbg4.py 8192x8192 0 2>&1 | tail -4
timeout 200 python scripts/dbg/c5dbg4.py 4096x4096 1 2>&1 | tail -4
