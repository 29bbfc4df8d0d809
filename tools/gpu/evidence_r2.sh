#!/bin/bash
# round-2 evidence: bench line (config 3, N = 33; cpu baseline, cold e2e), the
# reference arm, the ncu launch list of the bench, one full ncu capture of the
# specialised pass kernel (N = 28 config-3-recipe pass), per-target A timings.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev_smi.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo "ref exit $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-cold > gpurun_out/ev_ncu_bench.log 2>&1; echo "ncu list exit $?"
QSIM_LPASS_JIT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lpass_jit -s 2 -c 1 -f -o gpurun_out/ev_lpass python tools/prof_pass.py 28 2 > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full exit $?"
ncu -i gpurun_out/ev_lpass.ncu-rep --page raw --csv > gpurun_out/ev_lpass_raw.csv 2>&1
TARGETS=0,1,2,3,4,10,20,29 timeout 900 python tools/per_target.py A 30 10 > gpurun_out/ev_pt_a.json 2> gpurun_out/ev_pt_a.err; echo "per-target A exit $?"
tail -1 gpurun_out/ev_bench.json | cut -c1-300
