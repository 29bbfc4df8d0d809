mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_e.py -m gpu -x -q -k "remap" > gpurun_out/pytest_rp.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_rp.log
