#!/bin/bash
# config-5 QFT: per-pass HBM fraction at N=30/32, then ncu --set full of one specialised QFT pass at N=28
mkdir -p gpurun_out
export QSIM_LPASS_JIT=2
for n in 30 32; do timeout 600 python tools/prof_qft.py $n 3 > gpurun_out/qft_$n.json 2> gpurun_out/qft_$n.err; echo "qft $n rc=$?"; done
timeout 300 python tools/prof_qft.py 28 1 > gpurun_out/qft_28.json 2>&1; echo "plain 28 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lpass -s 3 -c 1 -f -o gpurun_out/qftpass python tools/prof_qft.py 28 1 > gpurun_out/ncu_qft.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/qftpass.ncu-rep --page raw --csv > gpurun_out/qftpass_raw.csv 2>&1
ncu -i gpurun_out/qftpass.ncu-rep --page details --csv > gpurun_out/qftpass_details.csv 2>&1
ncu -i gpurun_out/qftpass.ncu-rep --page source --csv --print-source sass > gpurun_out/qftpass_src.csv 2>&1
rm -f gpurun_out/qftpass.ncu-rep
ls -la gpurun_out | head -30
