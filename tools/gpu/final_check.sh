# full GPU suite + smoke + bench + latency, then the E tests with every pass specialised before first launch
bash tools/gpu/check_all.sh
QSIM_LPASS_JIT=2 timeout 900 python -m pytest tests/test_gpu_e.py -x -q -m gpu 2>&1 | tail -3
