# headline kernels of C1 / C3 / C4: one launch each under ncu --set full; export the raw page as CSV on the box
for spec in "c1:C1:gps:stream" "c3:C3:none:stream" "c4:C4:gps:stream-pull"; do
  IFS=: read tag cfg ro sched <<< "$spec"
  ncu --set full --clock-control none -k regex:hier_stream -s 1 -c 1 -o /tmp/prof_$tag python tools/prof_loop.py --config $cfg --reorder $ro --schedule $sched --runs 1 --timed 1 > /dev/null 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hier_stream|global_colour" --csv --log-file gpurun_out/launches_c1.csv python tools/prof_loop.py --config C1 --reorder gps --schedule stream --runs 2 --timed 1 > /dev/null 2>&1
ls -la gpurun_out
