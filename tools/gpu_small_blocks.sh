# small tiles: warp-sized CTAs make the colour barriers cheap (C5)
for spec in "structured:4,4 32" "structured:8,4 64" "structured:4,8 64" "gps 64" "gps 32" "structured:8,8 128"; do
  set -- $spec
  echo "=== C5 $1 block $2"
  timeout 600 python tools/prof_loop.py --config C5 --reorder $1 --block-size $2 --runs 3 --timed 7 --schedule stream,stream-pull,colour 2>&1 | grep -E "^hier|^blocks|Error|error" | cut -c1-300
done
for d in 3 4; do
  echo "=== depth $d C5 gps"
  MESHPLAN_STREAM_DEPTH=$d timeout 600 python tools/prof_loop.py --config C5 --reorder gps --runs 3 --timed 7 --schedule stream 2>&1 | grep -E "^hier|Error" | cut -c1-300
  echo "=== depth $d C5 structured:16,4"
  MESHPLAN_STREAM_DEPTH=$d timeout 600 python tools/prof_loop.py --config C5 --reorder structured:16,4 --runs 3 --timed 7 --schedule stream 2>&1 | grep -E "^hier|Error" | cut -c1-300
done
