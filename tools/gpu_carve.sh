# streamed executor: shared-memory carve-out (default / exact for the resident CTAs / max shared)
for cv in 0 1 100; do
  export MESHPLAN_STREAM_CARVEOUT=$cv
  timeout 300 python tools/prof_loop.py --config C5 --reorder gps --runs 3 --timed 9 --schedule stream 2>&1 | grep "^hier" | sed "s/^/carve=$cv C5 /"
  timeout 300 python tools/prof_loop.py --config C1 --reorder gps --runs 3 --timed 15 --schedule stream 2>&1 | grep "^hier" | sed "s/^/carve=$cv C1 /"
  timeout 300 python tools/prof_loop.py --config C3 --reorder none --runs 3 --timed 9 --schedule stream 2>&1 | grep "^hier" | sed "s/^/carve=$cv C3 /"
  timeout 600 python tools/prof_loop.py --config C4 --reorder structured:4,4,8 --block-size 480 --runs 3 --timed 9 --schedule stream,stream-pull 2>&1 | grep "^hier" | sed "s/^/carve=$cv C4s /"
done
