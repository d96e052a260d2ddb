set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench_c5.log
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 20 --cpu-seconds 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-600; done
