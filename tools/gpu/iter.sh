# one iteration: GPU tests, bench, ncu capture of the pass kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
QSIM_DEBUG_PASSES=1 timeout 120 python tools/prof_pass.py 30 20 > gpurun_out/passes.log 2>&1; echo "passes exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]);print('ms_per_step',d['ms_per_step'],'passes',d['library']['passes'],'roof',d['roofline']['bound'],d['roofline']['frac'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lpass_e -s 2 -c 1 -f -o gpurun_out/lpass python tools/prof_pass.py 28 2 > gpurun_out/ncu_lpass.log 2>&1; echo "ncu exit $?"
ncu -i gpurun_out/lpass.ncu-rep --page source --csv --print-source sass > gpurun_out/lpass_src.csv 2>&1
ncu -i gpurun_out/lpass.ncu-rep --page details --csv > gpurun_out/lpass_details.csv 2>&1
