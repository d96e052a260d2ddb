timeout 600 python tools/dag_stats.py --config C5 --lags 2048,4096,8192 2>&1 | grep lag
for ro in none cluster; do echo "=== C3 $ro"; timeout 900 python tools/prof_loop.py --config C3 --reorder $ro --runs 2 --timed 5 --schedule stream,colour,pipelined 2>&1 | grep -E "^hier|^blocks|^plan"; done
for ro in none gps; do echo "=== C2 $ro"; timeout 900 python tools/prof_loop.py --config C2 --reorder $ro --runs 2 --timed 5 --schedule stream,colour 2>&1 | grep -E "^hier|^blocks|^plan"; done
echo "=== C4 partition"; timeout 1500 python tools/prof_loop.py --config C4 --reorder partition --runs 2 --timed 5 --schedule stream,colour,pipelined 2>&1 | grep -E "^hier|^blocks|^plan"
