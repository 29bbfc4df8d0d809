# long random circuits vs the oracle: specialised kernels (QSIM_LPASS_JIT=2) and the interpreter (QSIM_LPASS_JIT=0)
mkdir -p gpurun_out
for m in 2 0; do
QSIM_LPASS_JIT=$m timeout 1500 python tools/stress_jit.py > gpurun_out/stress_jit_$m.json 2> gpurun_out/stress_jit_$m.err; echo "stress JIT=$m exit $?"
python -c "import json; d=json.load(open('gpurun_out/stress_jit_$m.json')); print('JIT=$m worst', d['worst'], 'jit_passes', sum(r['jit_passes'] for r in d['rows']), 'passes', sum(r['passes'] for r in d['rows']))"
done
