mkdir -p gpurun_out
timeout 600 python tools/xchg_loopback.py > gpurun_out/xchg_loopback.json 2> gpurun_out/xchg_loopback.err; echo "xl exit $?"; tail -5 gpurun_out/xchg_loopback.err
