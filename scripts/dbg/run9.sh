cd $GRAFT_REPO_ROOT
export ACA_SYNC_DEBUG=1
H='{"phys": {"beta": 0.4406868, "h": 0.0, "rule": 0, "init_q": 0.5}, "T": 20.0}'
for L in libvA.so libvB.so libvC.so; do echo $L; ACA_LIB=$L timeout 120 python scripts/dbg/c5dbg5.py 8192x8192 "$H"; done
