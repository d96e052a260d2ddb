# pull form with per-ref recomputation (no parking): parity and timing
MESHPLAN_PULL_RECOMPUTE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stream or executor" > gpurun_out/pytest_recompute.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_recompute.log
for rc in 0 1; do for spec in "C5 gps 128" "C5 structured:8,8 128" "C5 structured:16,4 128" "C5 structured:16,8 256" "C1 gps 128" "C4 partition 256"; do
  set -- $spec
  echo "=== recompute=$rc $1 $2 block $3"
  MESHPLAN_PULL_RECOMPUTE=$rc timeout 600 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 3 --timed 7 --schedule stream-pull 2>&1 | grep -E "^hier|Error|error" | cut -c1-300
done; done
MESHPLAN_PULL_RECOMPUTE=1 timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio --clock-control none -k regex:hier_stream -c 4 --csv python tools/prof_loop.py --config C5 --reorder structured:8,8 --schedule stream-pull --runs 1 --timed 1 > gpurun_out/ncu_recompute_8x8.csv 2>/dev/null; echo "ncu rc=$?"
