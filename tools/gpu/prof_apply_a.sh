mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_apply_a' -s 55 -c 1 -f -o gpurun_out/apply_a3 python tools/prof_pass.py 28 3 1 A > gpurun_out/ncu_a3.log 2>&1; echo "ncu exit $?"
ncu -i gpurun_out/apply_a3.ncu-rep --page source --csv --print-source sass > gpurun_out/apply_a3_src.csv 2>&1
ncu -i gpurun_out/apply_a3.ncu-rep --page details --csv > gpurun_out/apply_a3_details.csv 2>&1
