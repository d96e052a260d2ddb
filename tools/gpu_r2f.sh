# 256-bit increment-row accesses in the streamed executor: parity + C5/C1 timing; peer-exchange tests
timeout 1200 python -m pytest tests/test_decomp.py -x -q -m gpu -k "peer" > gpurun_out/pytest_peer.log 2>&1; echo "peer rc=$?"; tail -3 gpurun_out/pytest_peer.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stream or executor" > gpurun_out/pytest_row256.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_row256.log
for spec in "C5 gps 128" "C5 structured:8,8 128" "C5 structured:16,4 128" "C1 gps 128"; do
  set -- $spec
  echo "=== $1 $2 block $3"
  timeout 600 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 3 --timed 9 --schedule stream,stream-pull 2>&1 | grep -E "^hier|^blocks|Error|error" | cut -c1-300
done
timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum --clock-control none -k regex:hier_stream -c 5 --csv python tools/prof_loop.py --config C5 --reorder gps --schedule stream --runs 1 --timed 1 > gpurun_out/ncu_row256_gps.csv 2>/dev/null; echo "ncu rc=$?"
