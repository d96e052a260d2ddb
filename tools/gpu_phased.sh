timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for cfg in C5 C1 C2; do
  echo "=== $cfg"
  timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 7 --schedule stream 2>&1 | grep -E "^hier"
  MESHPLAN_STREAM_PER_COLOUR=1 timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 7 --schedule stream 2>&1 | grep -E "^hier" | sed 's/^/percolour /'
done
for cfg in C3; do echo "=== $cfg"; timeout 600 python tools/prof_loop.py --config $cfg --reorder none --runs 2 --timed 7 --schedule stream 2>&1 | grep -E "^hier"; 
  timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 7 --schedule stream 2>&1 | grep -E "^hier" | sed 's/^/gps /'; done
for cfg in C4; do echo "=== $cfg"; timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 7 --schedule stream 2>&1 | grep -E "^hier"; done
