timeout 900 python -m pytest tests -x -q -m gpu -k "random_data_many_blocks or medium or reference_plan or repeated" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
for cfg in C5 C1 C2; do
  echo "=== $cfg"
  timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 5 \
     --schedule stream,stream-dataflow --lags 1024,2048,3072,4096,8192 2>&1 | grep -E "^hier"
done
MESHPLAN_STREAM_STATS=1 timeout 600 python tools/prof_loop.py --config C5 --reorder gps --runs 2 --timed 3 \
     --schedule stream-dataflow --lags 1024,2048,3072,4096 2>&1 | grep -E "stats" | awk 'NR%5==0'
