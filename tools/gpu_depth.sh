# ring depth / resident CTAs on the latency-bound small loops (and C5)
for d in 2 3 4; do
  for c in C1 C2 C3 C5; do
    r=gps; [ $c = C3 ] && r=none
    MESHPLAN_STREAM_DEPTH=$d timeout 300 python tools/prof_loop.py --config $c --reorder $r --runs 3 --timed 15 --schedule stream 2>&1 | grep "^hier" | sed "s/^/depth=$d $c /"
  done
done
