mkdir -p gpurun_out
QSIM_LPASS_JIT=2 timeout 1500 python tools/stress_jit.py > gpurun_out/stress_jit.json 2> gpurun_out/stress_jit.err; echo "stress exit $?"; tail -20 gpurun_out/stress_jit.err; python -c "import json; print('worst', json.load(open('gpurun_out/stress_jit.json'))['worst'])"
