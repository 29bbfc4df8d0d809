# ncu capture of one specialised pass kernel (N=28, config-2 recipe, 2 layers)
mkdir -p gpurun_out
export QSIM_LPASS_JIT=2
timeout 300 python tools/prof_pass.py 28 2 > gpurun_out/prof_plain.log 2>&1; echo "plain exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lpass_jit -s 2 -c 1 -f -o gpurun_out/jit python tools/prof_pass.py 28 2 > gpurun_out/ncu_jit.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_jit.log
ncu -i gpurun_out/jit.ncu-rep --page raw --csv > gpurun_out/jit_raw.csv 2>&1
ncu -i gpurun_out/jit.ncu-rep --page source --csv --print-source sass > gpurun_out/jit_src.csv 2>&1
ncu -i gpurun_out/jit.ncu-rep --page details --csv > gpurun_out/jit_details.csv 2>&1
