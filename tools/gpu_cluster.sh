# the parallel GPU blocking (reorder="cluster") vs the bit-exact k-way partition: plan time, plan shape, loop time
for spec in "C4 256" "C4 128" "C1 128" "C5 128"; do
  set -- $spec
  for r in cluster partition; do
    if [ $1 = C5 ] && [ $r = partition ]; then continue; fi
    timeout 900 python tools/prof_loop.py --config $1 --reorder $r --block-size $2 --runs 3 --timed 9 --schedule stream,stream-pull,pipelined,pipelined-pull 2>&1 | grep "^hier\|^blocks\|^plan\|Error" | sed "s/^/$1 $r $2 /"
  done
done
