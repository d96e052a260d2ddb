for c in 0 4 5 6; do
  echo "== ctas=$c"
  MESHPLAN_STREAM_CTAS=$c timeout 600 python tools/prof_loop.py --config C5 --reorder gps --runs 2 --timed 5 \
     --schedule stream,stream-dataflow --lags 8192 2>&1 | grep -E "^hier"
done
