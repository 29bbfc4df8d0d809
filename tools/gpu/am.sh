mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_e.py -m gpu -x -q -k "apply_matrix" > gpurun_out/pytest_am.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_am.log
