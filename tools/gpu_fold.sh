#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fold2
python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "pencil" > gpurun_out/fold2/t_pencil.log 2>&1; echo "rc=$?" >> gpurun_out/fold2/t_pencil.log
# one-rank pencil through torchrun at 1024^3 (plain vs folded), peer and nccl
for x in peer nccl; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 1 --pgrid 1x1 --xchg $x --steps 10 --warmup 3 --no-e2e > gpurun_out/fold2/pencil1_plain_$x.json 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 1 --pgrid 1x1 --fold --xchg $x --steps 10 --warmup 3 --no-e2e > gpurun_out/fold2/pencil1_fold_$x.json 2>&1
done
