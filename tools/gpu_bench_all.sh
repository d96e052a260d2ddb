# one bench line per config (profiles/r02/bench_C*.json)
for c in C5 C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
