# block-size x schedule x lag sweep on C5 and C1 (GPS blocks)
for cfg in C1 C5; do
 for bs in 128 256 512; do
  echo "=== $cfg bs=$bs"
  timeout 600 python tools/prof_loop.py --config $cfg --reorder gps --block-size $bs --runs 3 --timed 7 \
     --schedule colour,pipelined,pipelined-pull,dataflow,pipelined-dataflow --lags 256,1024,4096,16384 2>&1 | grep -vi warn
 done
done
