mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_e.py -m gpu -x -q > gpurun_out/pytest_d1.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_d1.log
timeout 600 python tools/configs_1gpu.py cfg5_n32 cfg3_n33 s1_hwall > gpurun_out/configs_d1.json 2> gpurun_out/configs_d1.err; echo "cfg exit $?"; grep -E "cfg|s1" gpurun_out/configs_d1.err | cut -c1-170
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_d1.json 2> gpurun_out/bench_d1.err; echo "bench exit $?"
python -c "import json;d=json.loads(open('gpurun_out/bench_d1.json').read().splitlines()[-1]);print('ms_per_step',d['ms_per_step'],d['library']['passes'],d['roofline']['frac'])"
