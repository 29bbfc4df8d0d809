mkdir -p gpurun_out
QSIM_LPASS_K=11 timeout 600 python -m pytest tests/test_gpu_e.py -x -q > gpurun_out/pytest_k11.log 2>&1; echo "pytest k11 exit $?"; tail -2 gpurun_out/pytest_k11.log
run() { env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print('$*', 'ms_per_step %.1f'%d['ms_per_step'], 'passes', d['library']['passes'])"; }
run QSIM_LPASS_K=12
run QSIM_LPASS_K=11
