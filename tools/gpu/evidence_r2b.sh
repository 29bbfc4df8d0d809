#!/bin/bash
# round-2 evidence refresh after the A-kernel and persistent-kernel work
bash tools/gpu/evidence_r2.sh
timeout 900 python tools/configs_1gpu.py cfg4_n33 cfg4_lazy table4_adder > gpurun_out/ev_cfg.log 2>&1; echo "configs exit $?"
timeout 300 python tools/latency_cfg1.py 200 > gpurun_out/ev_latency.json 2> gpurun_out/ev_latency.err; echo "latency exit $?"
timeout 300 python tools/persist_sweep.py > gpurun_out/ev_persist.log 2>&1; echo "persist exit $?"
