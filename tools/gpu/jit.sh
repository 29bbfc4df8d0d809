mkdir -p gpurun_out
QSIM_LPASS_JIT_LOG=1 timeout 900 python -m pytest tests/test_gpu_e.py -m gpu -x -q -k "specialised or config2 or fused or config1" > gpurun_out/pytest_jit.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_jit.log
QSIM_LPASS_JIT_LOG=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_jit.json 2> gpurun_out/bench_jit.err; echo "bench exit $?"; tail -3 gpurun_out/bench_jit.err
python -c "import json;d=json.loads(open('gpurun_out/bench_jit.json').read().splitlines()[-1]);print('ms_per_step',d['ms_per_step'],'passes',d['library'],'roof',d['roofline']['bound'],d['roofline']['frac'])"
