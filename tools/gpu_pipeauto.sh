# warp-specialised executor: automatic ring depth / CTAs under a shared-memory budget per SM
export MESHPLAN_PIPE_VERBOSE=1
for kb in 192 160 228; do
  for spec in "C4 partition 256" "C4 structured:4,4,8 480" "C4 partition 128" "C1 gps 128" "C3 none 128"; do
    set -- $spec
    MESHPLAN_PIPE_SMEM_KB=$kb timeout 600 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 2 --timed 9 --schedule pipelined-pull,pipelined 2>&1 | grep "^hier\|^\[pipe\]" | sort -u | sed "s/^/kb=$kb $1 $2 $3 /"
  done
done
timeout 900 python -m pytest tests -m gpu -q -x -k "pipe or pipelined" 2>&1 | tail -2
