mkdir -p gpurun_out
timeout 1500 python tools/configs_1gpu.py > gpurun_out/configs_all.json 2> gpurun_out/configs_all.err; echo "cfg exit $?"; grep -E "^(cfg|s1|s2)" gpurun_out/configs_all.err | cut -c1-200
