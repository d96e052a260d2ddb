# row placement (bank groups): parity with it on, C5 tiles / GPS timing on vs off, bank conflicts; peer exchange tests
timeout 1200 python -m pytest tests/test_decomp.py -x -q -m gpu -k "peer" > gpurun_out/pytest_peer.log 2>&1; echo "peer rc=$?"; tail -3 gpurun_out/pytest_peer.log
MESHPLAN_ROW_PLACEMENT=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu -k "not c4_headline" > gpurun_out/pytest_placement.log 2>&1; echo "placement parity rc=$?"; tail -3 gpurun_out/pytest_placement.log
for pl in 0 1; do for spec in "gps 128" "structured:8,8 128" "structured:16,4 128" "structured:16,8 256"; do
  set -- $spec
  echo "=== placement=$pl C5 $1 block $2"
  MESHPLAN_ROW_PLACEMENT=$pl timeout 600 python tools/prof_loop.py --config C5 --reorder $1 --block-size $2 --runs 2 --timed 5 \
      --schedule stream,stream-pull,pipelined-pull,colour 2>&1 | grep -E "^hier|^blocks|Error|error" | cut -c1-300
done; done
MESHPLAN_ROW_PLACEMENT=1 timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:hier_stream -c 8 --csv python tools/prof_loop.py --config C5 --reorder structured:8,8 --schedule stream --runs 1 --timed 1 > gpurun_out/ncu_placed_8x8.csv 2>/dev/null; echo "ncu rc=$?"
