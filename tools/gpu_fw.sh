timeout 900 python -m pytest tests -x -q -m gpu -k "random_data_many_blocks or medium or reference_plan or structured or tma" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
for cfg in C5 C1 C2; do
  echo "=== $cfg"
  timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 5 --schedule stream 2>&1 | grep -E "^hier"
  timeout 600 python tools/prof_loop.py --config $cfg --reorder structured:16,4 --runs 2 --timed 5 --schedule stream 2>&1 | grep -E "^hier" | sed 's/^/struct /'
done
timeout 600 python tools/prof_loop.py --config C3 --reorder none --runs 2 --timed 5 --schedule stream,colour 2>&1 | grep -E "^hier" | sed 's/^/C3 /'
