# C5 higher-reuse blockings with the pull-form executors (2 barriers per block)
for r in structured:16,4 structured:8,8 gps; do
  timeout 600 python tools/prof_loop.py --config C5 --reorder $r --runs 3 --timed 9 --schedule stream,stream-pull,pipelined-pull 2>&1 | grep "^hier\|^blocks\|Error" | sed "s/^/$r /"
done
