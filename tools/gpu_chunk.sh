timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu --timeout 300 > gpurun_out/chunk_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/chunk_tests.log
for i in 1 2; do
timeout 300 python tools/prof_loop.py --config C5 --reorder gps --runs 3 --timed 10 --schedule stream 2>&1 | grep -E "^hier"
timeout 300 python tools/prof_loop.py --config C3 --reorder none --runs 3 --timed 10 --schedule stream,colour 2>&1 | grep -E "^hier"
done
timeout 300 python tools/prof_loop.py --config C4 --reorder partition --runs 3 --timed 10 --schedule stream,stream-pull 2>&1 | grep -E "^hier"
timeout 300 python tools/prof_loop.py --config C1 --reorder gps --runs 3 --timed 20 --schedule stream 2>&1 | grep -E "^hier"
