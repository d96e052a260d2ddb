# DRAM bytes per loop execution of each config's headline executor (ncu launch lists)
run() {  # config reorder schedule kernel-regex
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"$4" --csv --log-file gpurun_out/traffic_$1.csv \
    python tools/prof_loop.py --config $1 --reorder $2 --schedule $3 --runs 1 --timed 1 > gpurun_out/traffic_$1.log 2>&1
  echo "$1 rc=$?"
}
run C1 gps stream hier_stream
run C2 gps stream hier_stream
run C3 none stream hier_stream
run C4 partition pipelined-pull hier_pipe
