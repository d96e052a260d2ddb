# counters behind the pipe executor's shared-memory budget: one C4 k-way colour launch at 192 KB vs 228 KB per SM
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
for kb in 192 228; do
  MESHPLAN_PIPE_SMEM_KB=$kb MESHPLAN_PIPE_VERBOSE=1 timeout 900 ncu --metrics $M --clock-control none -k regex:hier_pipe_kernel --launch-skip 30 --launch-count 1 --csv --log-file gpurun_out/pipe_l1_$kb.csv python tools/prof_loop.py --config C4 --reorder partition --block-size 256 --runs 2 --timed 1 --schedule pipelined-pull > gpurun_out/pipe_l1_$kb.log 2>&1
  echo "kb=$kb rc=$?"
done
