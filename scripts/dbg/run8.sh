cd $GRAFT_REPO_ROOT
export ACA_SYNC_DEBUG=1
P="timeout 120 python scripts/dbg/c5dbg5.py 8192x8192"
H='"phys": {"beta": 0.4406868, "h": 0.0, "rule": 0, "init_q": 0.5}, "T": 20.0'
$P "{$H, \"event_hash\": 0}"
$P "{$H, \"max_ctas\": 74}"
$P "{$H, \"max_ctas\": 140}"
$P "{$H, \"rounds_per_launch\": 2}"
$P "{$H, \"rounds_per_launch\": 3}"
$P "{$H, \"tile\": [64, 32]}"
$P "{$H, \"tile\": [32, 32]}"
$P "{$H, \"seed\": 7}"
