cd $GRAFT_REPO_ROOT
timeout 200 python scripts/dbg/c5dbg2.py 8192x8192 1 10,50,100,150,200
timeout 200 python scripts/dbg/c5dbg2.py 8192x8192 0 10,50,100,200
timeout 200 python scripts/dbg/c5dbg2.py 2048x2048 1 50,100,150,200,300
timeout 200 python scripts/dbg/c5dbg2.py 8192x8192 1 200
