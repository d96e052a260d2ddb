# staged lists as id runs: GPU suite, then C5/C1/C2 with and without the run descriptors
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for rep in 1 2; do
for e in 1 0; do
  export MESHPLAN_STAGED_RUNS=$e
  timeout 300 python tools/prof_loop.py --config C5 --reorder gps --runs 3 --timed 9 --schedule stream 2>&1 | grep "^hier" | sed "s/^/runs=$e C5 /"
  timeout 300 python tools/prof_loop.py --config C1 --reorder gps --runs 3 --timed 15 --schedule stream 2>&1 | grep "^hier" | sed "s/^/runs=$e C1 /"
  timeout 300 python tools/prof_loop.py --config C2 --reorder gps --runs 3 --timed 15 --schedule stream 2>&1 | grep "^hier" | sed "s/^/runs=$e C2 /"
done
done
unset MESHPLAN_STAGED_RUNS
