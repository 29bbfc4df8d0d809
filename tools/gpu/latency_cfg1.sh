mkdir -p gpurun_out
timeout 300 python tools/latency_cfg1.py 200 > gpurun_out/latency_cfg1.json 2> gpurun_out/latency_cfg1.err; echo "lat exit $?"; tail -6 gpurun_out/latency_cfg1.err
QSIM_LPASS_JIT_MIN_TILES_LOG2=0 timeout 300 python tools/latency_cfg1.py 200 > gpurun_out/latency_cfg1_jit.json 2> gpurun_out/latency_cfg1_jit.err; echo "lat jit exit $?"; tail -6 gpurun_out/latency_cfg1_jit.err
