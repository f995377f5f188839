cd $GRAFT_REPO_ROOT
timeout 200 python scripts/dbg/c5dbg3.py 0
timeout 200 python scripts/dbg/c5dbg3.py 1
