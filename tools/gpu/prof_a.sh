# A-variant kernel timing (config-4 recipe, 1 GPU) and ncu captures of k_apply_a / k_bounds_a
mkdir -p gpurun_out
timeout 300 python tools/bench_kernels.py A 30 2 > gpurun_out/a_kernels.json 2> gpurun_out/a_kernels.err; echo "kernels exit $?"
python -c "
import json;d=json.loads(open('gpurun_out/a_kernels.json').read())
print('gates/s', d['gates_per_s'])
for k,v in d['kernels'].items(): print(k, v['launches'], '%.3f ms'%v['avg_ms'], '%.0f GB/s'%v['GBps'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_apply_a|k_bounds_a' -s 4 -c 2 -f -o gpurun_out/apply_a python tools/prof_pass.py 28 1 1 A > gpurun_out/ncu_a.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_a.log
ncu -i gpurun_out/apply_a.ncu-rep --page raw --csv > gpurun_out/apply_a_raw.csv 2>&1
ncu -i gpurun_out/apply_a.ncu-rep --page source --csv --print-source sass > gpurun_out/apply_a_src.csv 2>&1
ncu -i gpurun_out/apply_a.ncu-rep --page details --csv > gpurun_out/apply_a_details.csv 2>&1
