for st in all-indirect increment-only; do
  echo "=== C4 partition staging=$st"
  timeout 400 python tools/prof_loop.py --config C4 --reorder partition --staging $st --runs 2 --timed 8 --schedule stream,stream-pull 2>&1 | grep -E "^hier|^blocks"
  echo "=== C4 structured:4,4,8 bs480 staging=$st"
  timeout 400 python tools/prof_loop.py --config C4 --reorder structured:4,4,8 --block-size 480 --staging $st --runs 2 --timed 8 --schedule stream,stream-pull 2>&1 | grep -E "^hier|^blocks"
done
