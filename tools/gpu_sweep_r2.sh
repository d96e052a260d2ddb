# block-size sweeps: C4 k-way (the config's layout) and C1 GPS
for bs in 192 320 384; do
  echo "=== C4 partition block $bs"
  timeout 900 python tools/prof_loop.py --config C4 --reorder partition --block-size $bs --runs 2 --timed 5 \
      --schedule pipelined-pull,stream-pull,stream 2>&1 | grep -E "^hier|^blocks|Error|error" | cut -c1-300
done
for bs in 64 96 128 192; do
  echo "=== C1 gps block $bs"
  timeout 600 python tools/prof_loop.py --config C1 --reorder gps --block-size $bs --runs 3 --timed 9 \
      --schedule stream,colour 2>&1 | grep -E "^hier|^blocks|Error|error" | cut -c1-300
done
