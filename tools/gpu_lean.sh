#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/lean
for r in 1 2; do
python bench.py --n 1024 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/lean/lean1_$r.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/lean0/lib python bench.py --n 1024 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/lean/lean0_$r.json 2>&1
done
python tools/ab_summary.py gpurun_out/lean/*.json > gpurun_out/lean/summary.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/lean/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/lean/t_gpu.log
