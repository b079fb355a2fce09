# compute-sanitizer over scripts/sanitize.py: memcheck, racecheck (shared memory), synccheck
mkdir -p gpurun_out
T=${TAG:-san}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/${T}_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${T}_$tool.log
  tail -4 gpurun_out/${T}_$tool.log
done
# the whole GPU test suite (every ABI entry point, garden-size cases included) under memcheck
if [ -n "${SUITE}" ]; then
  timeout 2400 compute-sanitizer --tool memcheck --print-limit 30 --error-exitcode 9 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_memcheck_suite.log 2>&1
  echo "memcheck suite rc=$?" >> gpurun_out/${T}_memcheck_suite.log
  tail -6 gpurun_out/${T}_memcheck_suite.log
fi
# positive control: the tools must flag a planted out-of-bounds store and shared-memory race
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sanitizer_control scripts/sanitizer_control.cu
compute-sanitizer --tool memcheck /tmp/sanitizer_control > gpurun_out/${T}_control_memcheck.log 2>&1
compute-sanitizer --tool racecheck /tmp/sanitizer_control > gpurun_out/${T}_control_racecheck.log 2>&1
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/${T}_control_*.log
# racecheck / synccheck over the oracle-sized GPU tests (every ABI entry point; full-size cases excluded for time)
if [ -n "${RACE_SUITE}" ]; then
  for tool in racecheck synccheck; do
    timeout 2400 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 9 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py > gpurun_out/${T}_${tool}_suite.log 2>&1
    echo "$tool suite rc=$?" >> gpurun_out/${T}_${tool}_suite.log
    tail -4 gpurun_out/${T}_${tool}_suite.log
  done
fi
