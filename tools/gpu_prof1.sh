ncu --set full --clock-control none --import-source on -k regex:hier_pipe -s 1 -c 1 -o gpurun_out/prof_pipe_c5 \
  python tools/prof_loop.py --config C5 --reorder gps --schedule pipelined --runs 1 --timed 1 > gpurun_out/prof1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hier_block -s 1 -c 1 -o gpurun_out/prof_colour_c5 \
  python tools/prof_loop.py --config C5 --reorder gps --schedule colour --runs 1 --timed 1 >> gpurun_out/prof1.log 2>&1
