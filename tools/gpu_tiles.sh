# C5 quad tiles of growing size (reuse 3.05 -> 3.7) against the GPS headline, every colour schedule
for spec in "gps 128" "structured:8,8 128" "structured:16,8 256" "structured:16,16 512" "structured:32,16 1024" "structured:8,32 512"; do
  set -- $spec
  echo "=== C5 $1 block $2"
  timeout 600 python tools/prof_loop.py --config C5 --reorder $1 --block-size $2 --runs 2 --timed 5 \
      --schedule stream,stream-pull,pipelined,pipelined-pull,colour 2>&1 | grep -E "^hier|^blocks|^plan|Error|error" | cut -c1-400
done
