# structured (handcrafted) block-shape sweep on the hex configs
for sh in 4,4,8 8,4,4 2,8,8 8,8,2 4,8,4 2,4,16; do
  echo "=== C3 structured:$sh"
  timeout 600 python tools/prof_loop.py --config C3 --reorder structured:$sh --block-size 128 --runs 2 --timed 5 --schedule stream,stream-pull,colour 2>&1 | grep -E "^hier|^blocks"
done
for sh in 4,4,8 2,4,16 4,8,4 2,2,32; do
  echo "=== C4 structured:$sh (block 480)"
  timeout 600 python tools/prof_loop.py --config C4 --reorder structured:$sh --block-size 480 --runs 2 --timed 5 --schedule stream,stream-pull,pipelined,colour 2>&1 | grep -E "^hier|^blocks"
done
