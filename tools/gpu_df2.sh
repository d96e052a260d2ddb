timeout 900 python -m pytest tests -x -q -m gpu -k "random_data_many_blocks or medium or reference_plan" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
for cfg in C5 C1; do
  echo "=== $cfg"
  MESHPLAN_STREAM_STATS=1 timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 3 \
     --schedule stream,stream-dataflow --lags 2048,4096,8192,16384 2>&1 | grep -E "^hier|^blocks|stats" | tail -30
done
