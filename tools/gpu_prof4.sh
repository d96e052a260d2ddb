ncu --set full --clock-control none --import-source on -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_stream_c5_struct \
  python tools/prof_loop.py --config C5 --reorder structured:16,4 --schedule stream --runs 1 --timed 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_stream_c5_gps \
  python tools/prof_loop.py --config C5 --reorder gps --schedule stream --runs 1 --timed 1 > /dev/null 2>&1
