#!/bin/bash
# long random circuits vs the oracle with the bounds-checked specialised kernels (QSIM_LPASS_CHECK=1)
mkdir -p gpurun_out
QSIM_LPASS_JIT=2 QSIM_LPASS_CHECK=1 QSIM_JIT_DISK_CACHE=0 timeout 2400 python tools/stress_jit.py > gpurun_out/stress_check.json 2> gpurun_out/stress_check.err; echo "stress CHECK exit $?"
grep -c "lpass check failed" gpurun_out/stress_check.err
python -c "import json; d=json.load(open('gpurun_out/stress_check.json')); print('worst', d['worst'], 'jit_passes', sum(r['jit_passes'] for r in d['rows']), 'passes', sum(r['passes'] for r in d['rows']))"
