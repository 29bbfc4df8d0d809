mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_apply_a|k_bounds_a' -s 110 -c 2 -f -o gpurun_out/apply_a2 python tools/prof_pass.py 28 2 1 A > gpurun_out/ncu_a2.log 2>&1; echo "ncu exit $?"
tail -2 gpurun_out/ncu_a2.log
ncu -i gpurun_out/apply_a2.ncu-rep --page source --csv --print-source sass > gpurun_out/apply_a2_src.csv 2>&1
ncu -i gpurun_out/apply_a2.ncu-rep --page details --csv > gpurun_out/apply_a2_details.csv 2>&1
ncu -i gpurun_out/apply_a2.ncu-rep --page raw --csv > gpurun_out/apply_a2_raw.csv 2>&1
