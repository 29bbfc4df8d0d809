# round-end evidence: bench line, reference arm, ncu launch list + full capture, per-target E/A, the other configs
bash tools/gpu/evidence.sh
timeout 600 python tools/per_target.py E 30 10 > gpurun_out/re_per_target_E.json 2> gpurun_out/re_per_target_E.err; echo "pt E exit $?"
timeout 600 python tools/per_target.py A 30 10 > gpurun_out/re_per_target_A.json 2> gpurun_out/re_per_target_A.err; echo "pt A exit $?"
timeout 1500 python tools/configs_1gpu.py > gpurun_out/re_configs_all.json 2> gpurun_out/re_configs_all.err; echo "cfg exit $?"; grep -E "^(cfg|s1|s2)" gpurun_out/re_configs_all.err | cut -c1-200
