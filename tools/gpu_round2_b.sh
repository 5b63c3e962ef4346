#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_mgpu_gpu.py tests/test_headline_gpu.py -m gpu -x -q -s > gpurun_out/t_mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_mgpu.log
python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "slab or pencil" > gpurun_out/t_slab.log 2>&1; echo "rc=$?" >> gpurun_out/t_slab.log
# one-rank NCCL slab through torchrun: chunked vs whole-chunk exchange
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --slab --xchg nccl --steps 10 --warmup 3 --no-e2e > gpurun_out/slab1_chunked.json 2> gpurun_out/slab1_chunked.err
ARENA_SLAB_CHUNKS=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --slab --xchg nccl --steps 10 --warmup 3 --no-e2e > gpurun_out/slab1_whole.json 2> gpurun_out/slab1_whole.err
