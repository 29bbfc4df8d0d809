mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_a.py tests/test_gpu_asm.py -m gpu -x -q > gpurun_out/pytest_a3.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_a3.log
timeout 300 python tools/per_target.py A 30 10 > gpurun_out/per_target_A3.json 2> gpurun_out/per_target_A3.err; echo "pt A exit $?"; grep -E "t= (0|1|2|3|4|17|29) " gpurun_out/per_target_A3.err
timeout 600 python tools/configs_1gpu.py cfg4_trend cfg4_n33 s1_hwall > gpurun_out/configs_a3.json 2> gpurun_out/configs_a3.err; echo "cfg exit $?"; cat gpurun_out/configs_a3.err | tail -9
