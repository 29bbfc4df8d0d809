mkdir -p gpurun_out
timeout 600 python tools/per_target.py A 30 10 > gpurun_out/per_target_A4.json 2> gpurun_out/per_target_A4.err; echo "pt A exit $?"; grep -E "t= (0|4|17|29) " gpurun_out/per_target_A4.err
