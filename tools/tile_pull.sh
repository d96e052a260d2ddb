for sh in 16,4 8,8 32,2 8,4; do
  echo "=== C5 structured:$sh"
  timeout 400 python tools/prof_loop.py --config C5 --reorder structured:$sh --block-size 128 --runs 2 --timed 8 --schedule stream,stream-pull 2>&1 | grep -E "^hier|^blocks"
done
