mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_e.py -m gpu -x -q -k "shutdown" > gpurun_out/pytest_js.log 2>&1; echo "pytest exit $?"; tail -8 gpurun_out/pytest_js.log
