timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for cfg in C1 C5 C2 C3; do
  echo "=== $cfg"
  timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 3 --timed 7 \
     --schedule colour,pipelined,pipelined-dataflow,pipelined-dataflow-pull --lags 1024,2048,4096,8192 2>&1 | grep -E "^hier|^plan|^blocks"
done
