for sc in stream-pull stream; do
timeout 900 ncu --set full --clock-control none -k regex:hier_stream -s 5 -c 1 -o gpurun_out/prof_c4_$sc python tools/prof_loop.py --config C4 --reorder partition --schedule $sc --runs 1 --timed 1 > /dev/null 2>&1; echo "ncu $sc rc=$?"
ncu -i gpurun_out/prof_c4_$sc.ncu-rep --page raw --csv > gpurun_out/prof_c4_${sc}_raw.csv 2>/dev/null
rm -f gpurun_out/prof_c4_$sc.ncu-rep
done
