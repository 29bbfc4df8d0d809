mkdir -p gpurun_out
run() { env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v.json 2>gpurun_out/v.err; python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print('$*', 'ms_per_step %.1f'%d['ms_per_step'], d['library']['passes'])" || tail -3 gpurun_out/v.err; }
run LPASS_LOOKAHEAD=0
run LPASS_LOOKAHEAD=1 LPASS_FLIP_PENALTY=0
run LPASS_LOOKAHEAD=1 LPASS_FLIP_PENALTY=2
for la in 0 1; do LPASS_LOOKAHEAD=$la LPASS_FLIP_PENALTY=0 timeout 600 python tools/configs_1gpu.py cfg5_n32 cfg3_n33 2>&1 >/dev/null | grep -E "cfg" | sed "s/^/la=$la /"; done
