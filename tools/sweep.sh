#!/bin/bash
# Sensitivity sweep of the pipelined executor (stages x resident CTAs/SM) on one plan.
# usage: bash tools/sweep.sh C5 gps pipelined "2 3 4 6" "0 3 4 6 8"
CFG=${1:-C5}; REO=${2:-gps}; SCHED=${3:-pipelined}; STAGES=${4:-"2 3 4"}; CTAS=${5:-"0"}
for st in $STAGES; do
  for c in $CTAS; do
    echo "== stages=$st ctas=$c"
    MESHPLAN_PIPE_STAGES=$st MESHPLAN_PIPE_CTAS=$c python tools/prof_loop.py --config $CFG --reorder $REO \
      --schedule $SCHED --runs 2 --timed 5 2>&1 | grep -E "^hier|^global"
  done
done
