mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_fold.json 2> gpurun_out/bench_fold.err; echo "bench exit $?"
python -c "import json;d=json.loads(open('gpurun_out/bench_fold.json').read().splitlines()[-1]);print('ms_per_step',d['ms_per_step'],'passes',d['library']['passes'],'roof',d['roofline']['bound'],d['roofline']['frac'])"
