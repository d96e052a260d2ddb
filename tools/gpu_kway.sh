timeout 900 python -m pytest tests/test_gpu_kway.py tests/test_gpu_parity.py -q -x -m gpu -k "kway or matching or partition" > gpurun_out/kw_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/kw_tests.log
MESHPLAN_KWAY_TIMING=1 timeout 900 python tools/kway_time.py quad2d 5657,5657 flux > gpurun_out/kway_c5.log 2>&1; echo "c5 rc=$?"; grep -v Warn gpurun_out/kway_c5.log | tail -30
MESHPLAN_KWAY_TIMING=1 timeout 900 python tools/kway_time.py hex3d-faces 200,200,200 face-flux > gpurun_out/kway_c4.log 2>&1; echo "c4 rc=$?"; tail -3 gpurun_out/kway_c4.log
