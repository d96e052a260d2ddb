timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for cfg in C1 C5 C2 C3 C4; do
  echo "=== $cfg"
  for dep in 2 3; do
  MESHPLAN_STREAM_DEPTH=$dep timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 3 --timed 7 \
     --schedule colour,pipelined,stream,stream-dataflow --lags 2048,4096,8192 2>&1 | grep -E "^hier|^blocks" | sed "s/^/d$dep /"
  done
done
