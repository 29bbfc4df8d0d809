#!/bin/bash
mkdir -p gpurun_out
export QSIM_LPASS_JIT=2
timeout 300 python tools/prof_qft.py 28 1 > gpurun_out/qftp4_plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lpass -s 4 -c 1 -f -o gpurun_out/qftp4 python tools/prof_qft.py 28 1 > gpurun_out/ncu_qftp4.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/qftp4.ncu-rep --page raw --csv > gpurun_out/qftp4_raw.csv 2>&1
ncu -i gpurun_out/qftp4.ncu-rep --page source --csv --print-source sass > gpurun_out/qftp4_src.csv 2>&1
rm -f gpurun_out/qftp4.ncu-rep
