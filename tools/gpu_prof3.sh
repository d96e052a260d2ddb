for dep in 2 3 4; do
  echo "== depth=$dep"
  MESHPLAN_STREAM_DEPTH=$dep timeout 600 python tools/prof_loop.py --config C5 --reorder gps --runs 2 --timed 5 \
     --schedule stream,stream-dataflow --lags 8192 2>&1 | grep -E "^hier"
done
MESHPLAN_DATAFLOW_LAG=8192 ncu --set full --clock-control none --import-source on -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_streamdf_c5 \
  python tools/prof_loop.py --config C5 --reorder gps --schedule stream-dataflow --runs 1 --timed 1 > gpurun_out/prof3.log 2>&1
