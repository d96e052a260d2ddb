timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in C5 C1 C2; do for ro in gps structured:16,4; do
  [ "$c" = "C2" ] && [ "$ro" != "gps" ] && continue
  echo "=== $c $ro"; timeout 600 python tools/prof_loop.py --config $c --reorder $ro --runs 2 --timed 7 --schedule stream,stream-pull 2>&1 | grep -E "^hier"
done; done
echo "=== C3 none"; timeout 600 python tools/prof_loop.py --config C3 --reorder none --runs 2 --timed 7 --schedule stream,stream-pull 2>&1 | grep -E "^hier"
echo "=== C4 gps"; timeout 600 python tools/prof_loop.py --config C4 --reorder gps --runs 2 --timed 7 --schedule stream,stream-pull 2>&1 | grep -E "^hier"
echo "=== C4 cluster"; timeout 600 python tools/prof_loop.py --config C4 --reorder cluster --runs 2 --timed 7 --schedule stream,stream-pull 2>&1 | grep -E "^hier"
