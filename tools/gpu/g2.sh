mkdir -p gpurun_out
QSIM_LPASS_G2=1 timeout 600 python -m pytest tests/test_gpu_e.py -x -q > gpurun_out/pytest_g2.log 2>&1; echo "pytest g2 exit $?"; tail -2 gpurun_out/pytest_g2.log
run() { env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print('$*', 'ms_per_step %.1f'%d['ms_per_step'], 'passes', d['library']['passes'])"; }
run QSIM_LPASS_G2=0
run QSIM_LPASS_G2=1
QSIM_LPASS_G2=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lpass_e -s 2 -c 1 -f -o gpurun_out/lpass_g2 python tools/prof_pass.py 28 2 > gpurun_out/ncu_g2.log 2>&1; echo "ncu exit $?"
ncu -i gpurun_out/lpass_g2.ncu-rep --page source --csv --print-source sass > gpurun_out/lpass_g2_src.csv 2>&1
ncu -i gpurun_out/lpass_g2.ncu-rep --page details --csv > gpurun_out/lpass_g2_details.csv 2>&1
