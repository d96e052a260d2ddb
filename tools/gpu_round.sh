# full GPU round: tests, bench (all configs), launch list + ncu capture of the headline kernel
set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_C5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_C5.log | cut -c1-300
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 20 --cpu-seconds 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hier_stream|global_colour" -c 40 --csv --log-file gpurun_out/launches_c5.csv python tools/prof_loop.py --config C5 --reorder gps --schedule stream --runs 2 --timed 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hier_stream -s 2 -c 1 -o gpurun_out/prof_stream_c5 python tools/prof_loop.py --config C5 --reorder gps --schedule stream --runs 1 --timed 1 > /dev/null 2>&1; echo "ncu full rc=$?"
