mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_e.py -m gpu -x -q -k "specialised" > gpurun_out/pytest_jt.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_jt.log
