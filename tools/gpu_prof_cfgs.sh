# headline kernels of C1 / C3 / C4: one launch each under ncu --set full (source pages omitted to keep the files small)
ncu --set full --clock-control none -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_c1 python tools/prof_loop.py --config C1 --reorder gps --schedule stream --runs 1 --timed 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_c3 python tools/prof_loop.py --config C3 --reorder none --schedule stream --runs 1 --timed 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:hier_stream -s 1 -c 1 -o gpurun_out/prof_c4 python tools/prof_loop.py --config C4 --reorder gps --schedule stream-pull --runs 1 --timed 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hier_stream|global_colour" --csv --log-file gpurun_out/launches_c1.csv python tools/prof_loop.py --config C1 --reorder gps --schedule stream --runs 2 --timed 1 > /dev/null 2>&1
ls -la gpurun_out
