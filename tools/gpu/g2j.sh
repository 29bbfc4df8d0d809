mkdir -p gpurun_out
QSIM_LPASS_G=2 timeout 900 python -m pytest tests/test_gpu_e.py -m gpu -x -q -k "specialised" > gpurun_out/pytest_g2j.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_g2j.log
run() { env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v.json 2>gpurun_out/v.err; python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print('$*', 'ms_per_step %.1f'%d['ms_per_step'], d['library']['jit_passes'])" || tail -3 gpurun_out/v.err; }
run QSIM_LPASS_G=1
run QSIM_LPASS_G=2
