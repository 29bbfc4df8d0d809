#!/bin/bash
# one-GPU check of the torchrun / NCCL-transport plumbing of bench.py (BENCH_FORCE_DIST=1: one rank through
# the NCCL transport), and the reference arm under torchrun
mkdir -p gpurun_out
BENCH_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu --no-cold > gpurun_out/dist1.json 2> gpurun_out/dist1.err; echo "dist1 rc=$? stdout lines $(wc -l < gpurun_out/dist1.json)"; python -c "import json; d=json.load(open('gpurun_out/dist1.json')); print(d['ms_per_step'], d['config']['parallelism'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 1 --warmup 3 > gpurun_out/dist1_ref.json 2> gpurun_out/dist1_ref.err; echo "ref rc=$? stdout lines $(wc -l < gpurun_out/dist1_ref.json)"; python -c "import json; d=json.load(open('gpurun_out/dist1_ref.json')); print(d['impl'], d['value'])"
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 3 --no-cpu --no-cold > gpurun_out/gpus2.json 2> gpurun_out/gpus2.err; echo "gpus2 on one device rc=$?"; tail -3 gpurun_out/gpus2.err
