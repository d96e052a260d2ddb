# round 2: new GPU tests, the reference's own suite against this package, block-colouring timing
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python tools/reference_suite.py -- --tb=short -q -rf > gpurun_out/reference_suite.log 2>&1; echo "refsuite rc=$?"; tail -3 gpurun_out/reference_suite.log
timeout 900 python tools/time_block_colouring.py C1 C2 C3 C5 > gpurun_out/block_colouring_time.log 2>&1; echo "bc rc=$?"; cat gpurun_out/block_colouring_time.log | tail -5
