timeout 900 python -m pytest tests/test_decomp.py -x -q -m gpu -k "peer" > gpurun_out/pytest_peer.log 2>&1; echo "peer rc=$?"; tail -15 gpurun_out/pytest_peer.log
