#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/oop
for r in 1 2; do
python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/oop/plan_$r.json 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2953$r bench.py --gpus 1 --slab --xchg peer --steps 30 --warmup 5 --no-e2e > gpurun_out/oop/slab1peer_$r.json 2>&1
done
