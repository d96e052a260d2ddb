timeout 900 python -m pytest tests -x -q -m gpu -k "random_data_many_blocks or reference_plan or back_to_back" > gpurun_out/pytest_quick.log 2>&1; echo rc=$? >> gpurun_out/pytest_quick.log
timeout 600 python tools/prof_loop.py --config C5 --reorder gps --runs 2 --timed 7 --schedule stream,stream-dataflow --lags 4096,8192,65536 2>&1 | grep "^hier" > gpurun_out/dfo.log 2>&1
MESHPLAN_DATAFLOW_LAG=65536 ncu --set full --clock-control none --import-source on -k regex:hier_stream -s 1 -c 1 -o /tmp/p_df python tools/prof_loop.py --config C5 --reorder gps --schedule stream-dataflow --runs 1 --timed 1 > /dev/null 2>&1
ncu -i /tmp/p_df.ncu-rep --page raw --csv > gpurun_out/prof_df_raw.csv 2>/dev/null
ncu -i /tmp/p_df.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_df_src.csv 2>/dev/null
