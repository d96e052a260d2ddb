# automatic ring depth / CTAs (192 KB budget, two-CTA floor): parity, timings, C4 bench
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_decomp.py -m gpu -q -x 2>&1 | tail -2
export MESHPLAN_PIPE_VERBOSE=1
for spec in "C4 partition 256" "C4 structured:4,4,8 480" "C4 partition 128" "C1 gps 128" "C3 none 128"; do
  set -- $spec
  timeout 600 python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --runs 2 --timed 9 --schedule pipelined-pull,pipelined 2>&1 | grep "^hier\|^\[pipe\]" | sort -u | sed "s/^/auto $1 $2 $3 /"
done
unset MESHPLAN_PIPE_VERBOSE
timeout 900 python bench.py --config C4 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
