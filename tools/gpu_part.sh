echo "=== C4 partition"; timeout 1200 python tools/prof_loop.py --config C4 --reorder partition --runs 2 --timed 7 --schedule stream,stream-pull,pipelined,colour 2>&1 | grep -E "^hier|^blocks|^plan"
echo "=== C5 partition"; timeout 1500 python tools/prof_loop.py --config C5 --reorder partition --runs 2 --timed 7 --schedule stream,stream-pull,pipelined 2>&1 | grep -E "^hier|^blocks|^plan"
echo "=== C1 partition"; timeout 600 python tools/prof_loop.py --config C1 --reorder partition --runs 2 --timed 7 --schedule stream,stream-pull 2>&1 | grep -E "^hier|^blocks|^plan"
