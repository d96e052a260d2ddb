timeout 900 python -m pytest tests -x -q -m gpu -k "structured" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
for cfg in C5 C1; do for sh in 8,8 4,16 16,4; do
  echo "=== $cfg structured:$sh"
  timeout 900 python tools/prof_loop.py --config $cfg --reorder structured:$sh --runs 2 --timed 5 --schedule stream,pipelined,colour 2>&1 | grep -E "^hier|^blocks|^plan"
done; done
