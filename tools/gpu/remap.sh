mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_e.py tests/test_gpu_a.py -m gpu -x -q > gpurun_out/pytest_remap.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_remap.log
