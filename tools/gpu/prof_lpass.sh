# ncu capture of one k_lpass_e launch (N=28, config-2 recipe) + noio timing
mkdir -p gpurun_out
timeout 300 python tools/prof_pass.py 28 2 > gpurun_out/prof_plain.log 2>&1; echo "plain exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lpass_e -s 2 -c 1 -f -o gpurun_out/lpass python tools/prof_pass.py 28 2 > gpurun_out/ncu_lpass.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_lpass.log
ncu -i gpurun_out/lpass.ncu-rep --page raw --csv > gpurun_out/lpass_raw.csv 2>&1
ncu -i gpurun_out/lpass.ncu-rep --page source --csv --print-source sass > gpurun_out/lpass_src.csv 2>&1
ncu -i gpurun_out/lpass.ncu-rep --page details --csv > gpurun_out/lpass_details.csv 2>&1
ls -la gpurun_out
