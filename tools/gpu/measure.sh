# new GPU tests + §8(d) measurement rows (per-target, config-1 latency, per-GPU configs)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_e.py tests/test_gpu_a.py -m gpu -x -q -k "graph or overlap" > gpurun_out/pytest_new.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_new.log
timeout 300 python tools/per_target.py E 30 10 > gpurun_out/per_target_E.json 2> gpurun_out/per_target_E.err; echo "pt E exit $?"
timeout 300 python tools/per_target.py A 30 10 > gpurun_out/per_target_A.json 2> gpurun_out/per_target_A.err; echo "pt A exit $?"
timeout 300 python tools/latency_cfg1.py 200 > gpurun_out/latency_cfg1.json 2> gpurun_out/latency_cfg1.err; echo "lat exit $?"; cat gpurun_out/latency_cfg1.err | tail -8
timeout 900 python tools/configs_1gpu.py > gpurun_out/configs_1gpu.json 2> gpurun_out/configs_1gpu.err; echo "cfg exit $?"; cat gpurun_out/configs_1gpu.err | tail -12
