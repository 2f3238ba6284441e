set -e
cd $GRAFT_REPO_ROOT
python tools/profile_sweep.py --kind points3 --n 30000 --iters 3
LEANOT_GRAM=0 python tools/profile_sweep.py --kind points3 --n 30000 --iters 3
for g in 1 0; do
  LEANOT_GRAM=$g ncu --set full --import-source on --clock-control none -k regex:"rowpass|colpass" -s 2 -c 2 -o gpurun_out/pts_g$g -f python tools/profile_sweep.py --kind points3 --n 30000 --iters 3 > gpurun_out/ncu_g$g.log 2>&1
  ncu -i gpurun_out/pts_g$g.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread,smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__average_warp_latency_issue_stalled_lg_throttle,smsp__average_warp_latency_issue_stalled_math_pipe_throttle,smsp__average_warp_latency_issue_stalled_wait,smsp__average_warp_latency_issue_stalled_short_scoreboard,smsp__average_warp_latency_issue_stalled_not_selected,smsp__average_warp_latency_issue_stalled_dispatch_stall,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio > gpurun_out/pts_g$g.csv 2>&1
done
rm -f gpurun_out/*.ncu-rep
