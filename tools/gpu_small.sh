for c in C1 C2; do for bs in 64 96 128; do
  echo "=== $c bs=$bs"; timeout 600 python tools/prof_loop.py --config $c --reorder gps --block-size $bs --runs 3 --timed 9 --schedule stream 2>&1 | grep -E "^hier|^blocks"
done; done
for d in 3 4; do echo "=== C1 depth=$d"; MESHPLAN_STREAM_DEPTH=$d timeout 600 python tools/prof_loop.py --config C1 --reorder gps --runs 3 --timed 9 --schedule stream 2>&1 | grep -E "^hier"; done
