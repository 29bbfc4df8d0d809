mkdir -p gpurun_out
run() { env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v.json 2>gpurun_out/v.err; python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print('$*', 'ms_per_step %.1f'%d['ms_per_step'], d['library']['jit_passes'])" || tail -3 gpurun_out/v.err; }
run QSIM_LPASS_MINB=3
run QSIM_LPASS_MINB=2
