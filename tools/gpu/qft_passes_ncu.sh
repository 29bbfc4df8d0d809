#!/bin/bash
# per-launch duration / instructions / DRAM throughput of the 7 QFT passes at N=28 (one circuit, specialised kernels)
mkdir -p gpurun_out
export QSIM_LPASS_JIT=2
timeout 300 python tools/prof_qft.py 28 1 > gpurun_out/qftp_plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_sample_count --clock-control none -k regex:k_lpass --csv python tools/prof_qft.py 28 1 > gpurun_out/qft_passes_ncu.csv 2> gpurun_out/qft_passes_ncu.err; echo "ncu rc=$?"
