mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_a.py tests/test_gpu_asm.py -m gpu -x -q > gpurun_out/pytest_a4.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_a4.log
timeout 600 python tools/configs_1gpu.py cfg4_n33 > gpurun_out/configs_a4.json 2> gpurun_out/configs_a4.err; echo "cfg exit $?"; cat gpurun_out/configs_a4.err | tail -2
timeout 300 python tools/bench_kernels.py A 30 2 > gpurun_out/a_kernels.json 2> gpurun_out/a_kernels.err; echo "kernels exit $?"
python -c "
import json;d=json.loads(open('gpurun_out/a_kernels.json').read())
print('gates/s', d['gates_per_s'])
for k,v in d['kernels'].items(): print(k, v['launches'], '%.3f ms'%v['avg_ms'])"
