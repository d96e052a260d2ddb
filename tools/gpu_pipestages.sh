# warp-specialised executor: ring stages (shared bytes -> CTAs per SM) per plan
export MESHPLAN_PIPE_VERBOSE=1
for st in 2 3 4 5; do
  for spec in "C4 partition 256" "C4 structured:4,4,8 480" "C4 partition 128" "C1 gps 128" "C3 none 128" "C5 gps 128"; do
    set -- $spec
    MESHPLAN_PIPE_STAGES=$st timeout 600 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 2 --timed 9 --schedule pipelined-pull,pipelined 2>&1 | grep "^hier\|^\[pipe\]" | sort -u | sed "s/^/stages=$st $1 $2 $3 /"
  done
done
