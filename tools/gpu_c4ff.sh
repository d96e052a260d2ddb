# C4 k-way: block colours by the reference's least-loaded greedy vs first-fit (experiment)
for ch in least-loaded first-fit; do
  for bs in 256 480; do
  MESHPLAN_BLOCK_CHOOSER=$ch timeout 600 python tools/prof_loop.py --config C4 --reorder partition --block-size $bs --runs 3 --timed 9 --schedule stream,stream-pull,pipelined,pipelined-pull 2>&1 | grep "^hier\|^blocks\|Error" | sed "s/^/$ch $bs /"
  done
done
