# increment rows in shared memory (RSM) + register cap: main lib (RSM, cap 64),
# rsm72 (RSM, cap 72), norsm (registers, cap 72 = round-2 committed kernel)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py tests/test_gpu_configs.py -m gpu -x -q 2>&1 | tail -3
for v in main rsm72 norsm main rsm72 norsm; do
  if [ $v = main ]; then unset MESHPLAN_B200_LIB; else export MESHPLAN_B200_LIB=$PWD/paper_1802_03749_b200/lib/variants/libmeshplan_b200_$v.so; fi
  timeout 300 python tools/prof_loop.py --config C5 --reorder gps --runs 3 --timed 9 --schedule stream,stream-pull 2>&1 | grep "^hier" | sed "s/^/$v C5 /"
  timeout 300 python tools/prof_loop.py --config C1 --reorder gps --runs 3 --timed 9 --schedule stream 2>&1 | grep "^hier" | sed "s/^/$v C1 /"
  timeout 300 python tools/prof_loop.py --config C4 --reorder partition --block-size 256 --runs 3 --timed 9 --schedule stream,stream-pull 2>&1 | grep "^hier" | sed "s/^/$v C4 /"
done
unset MESHPLAN_B200_LIB
