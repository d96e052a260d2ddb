for cfg in C1 C5; do
 for ro in cluster; do
  for bs in 128 256; do
   echo "=== $cfg $ro bs=$bs"
   timeout 900 python tools/prof_loop.py --config $cfg --reorder $ro --block-size $bs --runs 2 --timed 5 \
     --schedule stream,pipelined,stream-dataflow --lags 8192 2>&1 | grep -E "^hier|^blocks|^plan"
  done
 done
done
echo "=== C1 partition"
timeout 900 python tools/prof_loop.py --config C1 --reorder partition --block-size 128 --runs 2 --timed 5 --schedule stream,pipelined,stream-dataflow --lags 8192 2>&1 | grep -E "^hier|^blocks|^plan"
timeout 900 python tools/prof_loop.py --config C1 --reorder partition --block-size 256 --runs 2 --timed 5 --schedule stream,pipelined --lags 8192 2>&1 | grep -E "^hier|^blocks|^plan"
