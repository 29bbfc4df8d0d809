# ncu --set full of one late-circuit k_bounds_a and k_apply_a (config-4 recipe, N=28)
mkdir -p gpurun_out
N=${1:-28}
python tools/a_cfg4_prof.py $N > gpurun_out/a_cfg4_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bounds_a|k_apply_a|k_p0tab' -s ${SKIP:-120} -c ${COUNT:-2} -f -o gpurun_out/a_dense_$N python tools/a_cfg4_prof.py $N > gpurun_out/ncu_a_dense.log 2>&1; echo "ncu exit $?"
ncu -i gpurun_out/a_dense_$N.ncu-rep --page details --csv > gpurun_out/a_dense_${N}_details.csv 2>&1
ncu -i gpurun_out/a_dense_$N.ncu-rep --page raw --csv > gpurun_out/a_dense_${N}_raw.csv 2>&1
ncu -i gpurun_out/a_dense_$N.ncu-rep --page source --csv --print-source sass > gpurun_out/a_dense_${N}_src.csv 2>&1
