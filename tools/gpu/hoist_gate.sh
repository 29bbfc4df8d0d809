#!/bin/bash
# the per-tile hoisting gated by tile count: checked kernels with it forced on / off, config-1 latency, QFT timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_e.py -q -m gpu -k "bounds_checked or phase_ops or variants" > gpurun_out/hg_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/hg_pytest.log
timeout 300 python tools/latency_cfg1.py 200 > gpurun_out/latency_cfg1.json 2> gpurun_out/latency_cfg1.err; echo "lat rc=$?"; tail -6 gpurun_out/latency_cfg1.err
export QSIM_LPASS_JIT=2
for n in 30 32; do timeout 600 python tools/prof_qft.py $n 3 > gpurun_out/qft_hoist_$n.json 2> gpurun_out/qft_hoist_$n.err; echo "qft $n rc=$? $(python -c "import json;d=json.load(open('gpurun_out/qft_hoist_$n.json'));print(round(d['ms_per_circuit_passes'],1),'ms',round(d['hbm_GBps_passes']),'GB/s')")"; done
