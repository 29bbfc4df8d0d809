mkdir -p gpurun_out
timeout 900 python tools/qft_full_check.py 30 > gpurun_out/qft_full.json 2> gpurun_out/qft_full.err; echo "qft exit $?"; cat gpurun_out/qft_full.json; tail -3 gpurun_out/qft_full.err
