timeout 900 python -m pytest tests -x -q -m gpu -k "random_data_many_blocks or medium or reference_plan" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
for ro in none gps; do echo "=== C3 $ro"; timeout 900 python tools/prof_loop.py --config C3 --reorder $ro --runs 2 --timed 5 --schedule stream,colour,pipelined 2>&1 | grep -E "^hier"; done
for ro in cluster gps; do echo "=== C4 $ro"; timeout 900 python tools/prof_loop.py --config C4 --reorder $ro --runs 2 --timed 5 --schedule stream,colour,pipelined 2>&1 | grep -E "^hier|^blocks"; done
