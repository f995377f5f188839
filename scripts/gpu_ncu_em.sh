# EM=1 (a10 only) vs EM=2 (a10 + class bookkeeping) on c5: instruction counts, issue, stalls
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ncuem}
M=smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
for CB in 0 1; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:tile_grp -s 40 -c 4 --csv python bench.py --config c5 --class-book $CB --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_em_cb${CB}_$TAG.csv 2> gpurun_out/ncu_em_cb${CB}_$TAG.err
  echo "cb=$CB rc=$?"
done
