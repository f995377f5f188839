cd $GRAFT_REPO_ROOT
timeout 120 python scripts/dbg/c5dbg.py 512x512 0 5 oracle; echo rc=$?
timeout 120 python scripts/dbg/c5dbg.py 512x512 2 5 oracle; echo rc=$?
timeout 120 python scripts/dbg/c5dbg.py 1024x1024 0 20; echo rc=$?
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python scripts/dbg/c5dbg.py 256x256 2 3 2>&1 | head -40; echo rc=$?
