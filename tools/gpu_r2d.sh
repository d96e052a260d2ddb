# ncu full captures of one colour launch: C5 GPS stream (headline) vs 8x8 tiles (stream, pipelined-pull);
# reports are exported to CSV on the box and deleted (gpurun_out must stay under 64 MiB)
for spec in "gps stream hier_stream" "structured:8,8 stream hier_stream" "structured:8,8 pipelined-pull hier_pipe"; do
  set -- $spec
  tag=$(echo $1 | tr ':,' '__')_$2
  rep=/tmp/r2_c5_$tag
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o $rep \
      python tools/prof_loop.py --config C5 --reorder $1 --schedule $2 --runs 1 --timed 1 > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/r2_c5_${tag}_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_c5_${tag}_sass.csv 2>/dev/null
  gzip -f gpurun_out/r2_c5_${tag}_sass.csv
  ls -la gpurun_out/r2_c5_${tag}*
done
timeout 1200 python -m pytest tests/test_decomp.py -x -q -m gpu -k "peer" > gpurun_out/pytest_peer.log 2>&1; echo "peer rc=$?"; tail -15 gpurun_out/pytest_peer.log
bash tools/race_control.sh
du -sh gpurun_out
