#!/bin/bash
# PHASES terms on full-index bits hoisted to one product per tile, conditional
# scalars on full-index bits applied at the tile store: E parity (interpreter +
# specialised, and every pass specialised), then QFT per-pass timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_e.py tests/test_gpu_adder.py tests/test_gpu_asm.py -x -q -m gpu > gpurun_out/hoist_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/hoist_pytest.log
QSIM_LPASS_JIT=2 timeout 900 python -m pytest tests/test_gpu_e.py tests/test_gpu_adder.py -x -q -m gpu > gpurun_out/hoist_pytest_jit.log 2>&1; echo "pytest jit rc=$?"; tail -2 gpurun_out/hoist_pytest_jit.log
export QSIM_LPASS_JIT=2
for n in 30 32; do timeout 600 python tools/prof_qft.py $n 3 > gpurun_out/qft_hoist_$n.json 2> gpurun_out/qft_hoist_$n.err; echo "qft $n rc=$? $(python -c "import json;d=json.load(open('gpurun_out/qft_hoist_$n.json'));print(round(d['ms_per_circuit_passes'],1),'ms',round(d['hbm_GBps_passes']),'GB/s')")"; done
