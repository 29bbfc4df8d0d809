# round evidence: bench line (+cpu baseline), reference arm, ncu launch list, full capture of the specialised pass kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev_smi.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ev_ncu_bench.log 2>&1; echo "ncu list exit $?"
QSIM_LPASS_JIT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lpass_jit -s 2 -c 1 -f -o gpurun_out/ev_lpass python tools/prof_pass.py 28 2 > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full exit $?"
ncu -i gpurun_out/ev_lpass.ncu-rep --page raw --csv > gpurun_out/ev_lpass_raw.csv 2>&1
ncu -i gpurun_out/ev_lpass.ncu-rep --page details --csv > gpurun_out/ev_lpass_details.csv 2>&1
tail -2 gpurun_out/ev_bench.json | cut -c1-400
