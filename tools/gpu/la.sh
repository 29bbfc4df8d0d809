mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print('$*', 'ms_per_step %.1f'%d['ms_per_step'], 'passes', d['library']['passes'])"; }
run LPASS_LOOKAHEAD=0
run LPASS_LOOKAHEAD=1 LPASS_FLIP_PENALTY=0
run LPASS_LOOKAHEAD=1 LPASS_FLIP_PENALTY=2
run LPASS_LOOKAHEAD=1 LPASS_FLIP_PENALTY=4
run LPASS_LOOKAHEAD=1 LPASS_FLIP_PENALTY=8
