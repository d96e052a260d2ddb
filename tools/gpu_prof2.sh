ncu --set full --clock-control none --import-source on -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_stream_c5 \
  python tools/prof_loop.py --config C5 --reorder gps --schedule stream --runs 1 --timed 1 > gpurun_out/prof2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_streamdf_c5 \
  python tools/prof_loop.py --config C5 --reorder gps --schedule stream-dataflow --runs 1 --timed 1 >> gpurun_out/prof2.log 2>&1
