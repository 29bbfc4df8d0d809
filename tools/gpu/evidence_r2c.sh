#!/bin/bash
# round-2 final evidence: the bench line + launch list + reference arm
# (evidence_r2.sh, which also runs per-target A with the default policy and
# the ncu pass capture), per-target A under the fp32 variant, the config-4 /
# adder rows, config-1 latency, the persistent-kernel sweep, and one ncu
# capture of the A dense kernels.
bash tools/gpu/evidence_r2.sh
A_POLICY=fp32 TARGETS=0,1,2,3,4,10,20,29 timeout 900 python tools/per_target.py A 30 10 > gpurun_out/ev_pt_a_fp32.json 2> gpurun_out/ev_pt_a_fp32.err; echo "per-target A fp32 exit $?"
timeout 1200 python tools/configs_1gpu.py cfg4_n33 cfg4_lazy table4_adder > gpurun_out/ev_cfg.log 2>&1; echo "configs exit $?"
timeout 300 python tools/latency_cfg1.py 200 > gpurun_out/ev_latency.json 2> gpurun_out/ev_latency.err; echo "latency exit $?"
timeout 300 python tools/persist_sweep.py > gpurun_out/ev_persist.log 2>&1; echo "persist exit $?"
bash tools/gpu/prof_a_dense.sh 28 > /dev/null 2>&1; echo "ncu A exit $?"
