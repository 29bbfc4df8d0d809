# bench variants of the pass kernel (ms per config-2 step)
mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print('$*', 'ms_per_step %.1f'%d['ms_per_step'], 'passes', d['library']['passes'])"; }
run QSIM_PASS_R=4
run QSIM_PASS_R=5
run QSIM_LPASS_NODEFER=1
run QSIM_PASS_KERNEL=0
