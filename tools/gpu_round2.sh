# round 2 measurement pass: every config's bench line, the reference arm, the N>1 rank path at world size 1,
# launch lists (ncu gpu__time_duration) and one ncu --set full capture per headline kernel (exported to CSV)
set -x
timeout 900 python bench.py > gpurun_out/bench_C5.log 2>&1; echo "bench C5 rc=$?"; tail -1 gpurun_out/bench_C5.log | cut -c1-300
for c in C1 C2 C3 C4; do timeout 900 python bench.py --config $c --steps 20 --cpu-seconds 5 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 tools/rank_smoke.py --config C5 --steps 10 > gpurun_out/rank_smoke_c5.log 2>&1; echo "rank smoke rc=$?"; tail -1 gpurun_out/rank_smoke_c5.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hier_stream|global_colour" -c 40 --csv python tools/prof_loop.py --config C5 --reorder gps --schedule stream --runs 2 --timed 1 > gpurun_out/launches_c5.csv 2>/dev/null; echo "ncu launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hier_pipe" -c 60 --csv python tools/prof_loop.py --config C4 --reorder partition --block-size 256 --schedule pipelined-pull --runs 2 --timed 1 > gpurun_out/launches_c4.csv 2>/dev/null; echo "ncu launches c4 rc=$?"
for spec in "C5 gps 128 stream hier_stream" "C4 partition 256 pipelined-pull hier_pipe" "C1 gps 128 stream hier_stream" "C3 none 128 stream hier_stream"; do
  set -- $spec
  rep=/tmp/r2full_$1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$5 -s 3 -c 1 -o $rep \
      python tools/prof_loop.py --config $1 --reorder $2 --block-size $3 --schedule $4 --runs 1 --timed 1 > /dev/null 2>&1
  echo "ncu full $1 rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/r2full_$1_raw.csv 2>/dev/null
done
du -sh gpurun_out
