mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_e.py -m gpu -x -q > gpurun_out/pytest_fold.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_fold.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_fold.json 2> gpurun_out/bench_fold.err; echo "bench exit $?"
python -c "import json;d=json.loads(open('gpurun_out/bench_fold.json').read().splitlines()[-1]);print('ms_per_step',d['ms_per_step'],'passes',d['library']['passes'],'roof',d['roofline']['bound'],d['roofline']['frac'])"
