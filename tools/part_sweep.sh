# k-way partition block-size sweep on C4 (face loop) and C3 (scatter8)
for bs in 64 128 256 512; do
  echo "=== C4 partition bs=$bs"
  timeout 600 python tools/prof_loop.py --config C4 --reorder partition --block-size $bs --runs 2 --timed 5 --schedule stream,stream-pull,pipelined,colour 2>&1 | grep -E "^hier|^blocks"
done
for bs in 128 256; do
  echo "=== C3 partition bs=$bs"
  timeout 600 python tools/prof_loop.py --config C3 --reorder partition --block-size $bs --runs 2 --timed 5 --schedule stream,stream-pull,colour 2>&1 | grep -E "^hier|^blocks"
done
