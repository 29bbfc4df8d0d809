mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; done; tail -2 gpurun_out/smoke.log
timeout 300 python tools/latency_cfg1.py 50 > /dev/null 2>&1; echo "lat exit $?"
