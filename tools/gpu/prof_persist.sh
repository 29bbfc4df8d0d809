# ncu --set full of one persistent-kernel launch (config 1, N=14)
mkdir -p gpurun_out
cat > /tmp/pp.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import paper_1805_04708_b200 as q, qsim_inputs as C
with q.State(14) as s:
    c = C.config(0, n=14, seed=0)
    s.apply_circuit_persistent(c); s.apply_circuit_persistent(c); s.sync()
PY
python /tmp/pp.py || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -f -o gpurun_out/persist14 python /tmp/pp.py > gpurun_out/ncu_persist.log 2>&1; echo "ncu exit $?"
ncu -i gpurun_out/persist14.ncu-rep --page raw --csv > gpurun_out/persist14_raw.csv 2>&1
ncu -i gpurun_out/persist14.ncu-rep --page source --csv --print-source sass > gpurun_out/persist14_src.csv 2>&1
