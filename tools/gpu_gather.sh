# gather-form executor: parity then timing vs the push form on the headline layouts
timeout 1200 python -m pytest tests/test_gpu_gather.py -x -q -m gpu > gpurun_out/pytest_gather.log 2>&1; echo "gather tests rc=$?"; tail -15 gpurun_out/pytest_gather.log
for spec in "C5 gps 128" "C5 structured:8,8 128" "C5 structured:16,4 128" "C5 structured:16,8 256" "C5 structured:16,16 480" "C1 gps 128" "C1 structured:8,8 128" "C3 none 128" "C4 partition 256" "C4 structured:4,4,8 480"; do
  set -- $spec
  echo "=== $1 $2 block $3"
  timeout 900 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 3 --timed 7 --schedule stream,gather 2>&1 | grep -E "^hier|^blocks|Error|error" | cut -c1-300
done
timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__block_size --clock-control none -k regex:hier_gather -c 4 --csv python tools/prof_loop.py --config C5 --reorder structured:8,8 --schedule gather --runs 1 --timed 1 > gpurun_out/ncu_gather_8x8.csv 2>/dev/null; echo "ncu rc=$?"
