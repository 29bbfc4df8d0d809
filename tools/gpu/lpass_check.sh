set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -25 gpurun_out/pytest_gpu.log
QSIM_DEBUG_PASSES=1 timeout 120 python tools/prof_pass.py 26 2 > gpurun_out/passes.log 2>&1; echo "passes exit $?"; head -20 gpurun_out/passes.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
for r in 5; do QSIM_PASS_R=$r timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r$r.json 2>&1; echo "bench R=$r exit $?"; python -c "import json;d=json.loads(open('gpurun_out/bench_r$r.json').read().splitlines()[-1]);print('R=$r ms_per_step',d['ms_per_step'])"; done
