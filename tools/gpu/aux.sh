mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_aux.py tests/test_abi.py -q > gpurun_out/pytest_aux.log 2>&1; echo "pytest aux exit $?"; tail -3 gpurun_out/pytest_aux.log
timeout 300 python tools/bench_aux.py 36 24 64 > gpurun_out/bench_aux.json 2>&1; echo "bench_aux exit $?"; cat gpurun_out/bench_aux.json
timeout 300 python tools/bench_aux.py 36 28 16 >> gpurun_out/bench_aux.json 2>&1; tail -1 gpurun_out/bench_aux.json
