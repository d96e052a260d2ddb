timeout 900 python -m pytest tests/test_reference_suite.py tests/test_plan_interop.py -x -q -m gpu > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2c.log
bash tools/gpu_tiles.sh > gpurun_out/tiles.log 2>&1; echo "tiles rc=$?"; cat gpurun_out/tiles.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-seconds 3 > gpurun_out/bench_C5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_C5.log | cut -c1-200
