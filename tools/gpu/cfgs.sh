mkdir -p gpurun_out
timeout 1200 python tools/configs_1gpu.py cfg3_n33 cfg5_n32 s1_hwall s2_ghz > gpurun_out/configs_e.json 2> gpurun_out/configs_e.err; echo "cfg exit $?"; cat gpurun_out/configs_e.err | tail -8
