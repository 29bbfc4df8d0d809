#!/bin/bash
# compute-sanitizer over the small workload (tools/sanitize_small.py): one tool
# per pass -- memcheck, racecheck (shared-memory hazards of the tile pass and
# the A kernels), synccheck -- with the specialised pass kernels compiled
# before their first launch so they are what runs.
mkdir -p gpurun_out
export QSIM_LPASS_JIT=2
python tools/sanitize_small.py > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/san_plain.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tail -2 | tr '\n' ' ')"
done
