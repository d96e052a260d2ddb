# C4 (k-way partition, staged reads): pipelined stages / stream depth sweeps
for st in 2 3 4 5; do echo "=== pipe stages $st"; MESHPLAN_PIPE_STAGES=$st timeout 400 python tools/prof_loop.py --config C4 --reorder partition --runs 2 --timed 8 --schedule pipelined-pull,pipelined 2>&1 | grep -E "^hier"; done
for d in 2 3 4; do echo "=== stream depth $d"; MESHPLAN_STREAM_DEPTH=$d timeout 400 python tools/prof_loop.py --config C4 --reorder partition --runs 2 --timed 8 --schedule stream,stream-pull 2>&1 | grep -E "^hier"; done
for bs in 64 96; do echo "=== bs $bs"; timeout 400 python tools/prof_loop.py --config C4 --reorder partition --block-size $bs --runs 2 --timed 8 --schedule pipelined-pull,stream 2>&1 | grep -E "^hier|^blocks"; done
