cd $GRAFT_REPO_ROOT
export ACA_SYNC_DEBUG=1
H='{"phys": {"beta": 0.4406868, "h": 0.0, "rule": 0, "init_q": 0.5}, "T": 20.0}'
for L in libvF.so libvG.so libvH.so; do echo $L; ACA_LIB=$L timeout 100 python scripts/dbg/c5dbg5.py 8192x8192 "$H"; ACA_LIB=$L timeout 100 python scripts/dbg/c5dbg5.py 8192x8192 '{"rounds_per_launch": 8}'; done
