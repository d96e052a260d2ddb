# C4 (face flux, k-way partition = the config's named layout) at larger block sizes
for bs in 256 480; do
  echo "=== C4 partition block $bs"
  timeout 900 python tools/prof_loop.py --config C4 --reorder partition --block-size $bs --runs 2 --timed 5 \
      --schedule pipelined-pull,pipelined,stream-pull,stream,colour 2>&1 | grep -E "^hier|^blocks|^plan|Error|error" | cut -c1-300
done
