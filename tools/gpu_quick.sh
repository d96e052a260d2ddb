# quick: parity subset + stream timings
timeout 900 python -m pytest tests -x -q -m gpu -k "random_data_many_blocks or medium or reference_plan" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
for cfg in ${CFGS:-C1 C5}; do
  echo "=== $cfg"
  for dep in ${DEPS:-2 3}; do
  MESHPLAN_STREAM_DEPTH=$dep timeout 600 python tools/prof_loop.py --config $cfg --reorder ${REORDER:-gps} --runs 3 --timed 7 \
     --schedule ${SCHEDS:-stream,stream-dataflow} --lags ${LAGS:-4096} 2>&1 | grep -E "^hier|^blocks" | sed "s/^/d$dep /"
  done
done
