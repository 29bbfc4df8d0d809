# stage accesses as explicit 16-byte shared loads/stores: parity, bench, one full capture of a config-2-like pass
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_e.py -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/lds_bench.json 2> gpurun_out/lds_bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('gpurun_out/lds_bench.json').read().strip().splitlines()[-1]); print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], d['clocks'])"
QSIM_LPASS_JIT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lpass_jit -s 5 -c 1 -f -o gpurun_out/lds_lpass python tools/prof_pass.py 28 20 > gpurun_out/lds_ncu.log 2>&1; echo "ncu full exit $?"
ncu -i gpurun_out/lds_lpass.ncu-rep --page raw --csv > gpurun_out/lds_lpass_raw.csv 2>&1
