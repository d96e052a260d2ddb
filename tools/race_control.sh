# racecheck negative / positive controls for hier_pipe_kernel (warp-specialised executor):
#   shipped  -- the production library
#   ctl1     -- MP_PIPE_RACE_CONTROL=1: producer skips the empty-barrier wait (a real stage-reuse race)
#   ctl2     -- MP_PIPE_RACE_CONTROL=2: cp.async.wait_all + plain mbarrier.arrive instead of arrive.noinc
# libraries built in the build container: python -c "from paper_1802_03749_b200 import build_native as b; b.build(defines=['MP_PIPE_RACE_CONTROL=1'], tag='ctl1')"
for v in shipped ctl1 ctl2; do
  if [ $v = shipped ]; then unset MESHPLAN_B200_LIB; else export MESHPLAN_B200_LIB=$PWD/paper_1802_03749_b200/lib/variants/libmeshplan_b200_$v.so; fi
  echo "== $v: racecheck over pipelined, pipelined-pull"
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize.py pipelined,pipelined-pull > gpurun_out/race_$v.log 2>&1
  grep -E "RACECHECK SUMMARY|sanitize run ok" gpurun_out/race_$v.log
  grep -oE "(Read-after-Write|Write-after-Read|Write-after-Write) hazard" gpurun_out/race_$v.log | sort | uniq -c
  echo "== $v: executor parity (pipelined schedules, golden cases)"
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "executor_on_reference_plan" -x > gpurun_out/race_tests_$v.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/race_tests_$v.log
done
