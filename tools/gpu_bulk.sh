# read rows through per-lane TMA bulk copies (MESHPLAN_STREAM_BULK=1) vs LDGSTS: parity and timing
MESHPLAN_STREAM_BULK=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stream or executor" > gpurun_out/pytest_bulk.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_bulk.log
for b in 0 1; do for spec in "C5 gps 128" "C5 structured:8,8 128" "C1 gps 128"; do
  set -- $spec
  echo "=== bulk=$b $1 $2 block $3"
  MESHPLAN_STREAM_BULK=$b timeout 600 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 3 --timed 9 --schedule stream,stream-pull 2>&1 | grep -E "^hier|Error|error" | cut -c1-300
done; done
MESHPLAN_STREAM_BULK=1 timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:hier_stream -c 5 --csv python tools/prof_loop.py --config C5 --reorder gps --schedule stream --runs 1 --timed 1 > gpurun_out/ncu_bulk_gps.csv 2>/dev/null; echo "ncu rc=$?"
for spec in "C2 gps 64" "C2 gps 96" "C2 none 128" "C2 none 256" "C3 none 64" "C3 none 96"; do
  set -- $spec
  echo "=== $1 $2 block $3"
  timeout 600 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 3 --timed 9 --schedule stream,colour,stream-dataflow 2>&1 | grep -E "^hier|^blocks|Error|error" | cut -c1-300
done
