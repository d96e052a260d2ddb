timeout 900 python -m pytest tests/test_decomp.py tests/test_gpu_parity.py -x -q -m gpu -k "peer or executor or stream" > gpurun_out/pytest_check.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_check.log
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_C5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_C5.log | cut -c1-300
