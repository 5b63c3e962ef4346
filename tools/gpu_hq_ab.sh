#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab3
python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "quadrant or repeat" > gpurun_out/ab3/t_hq.log 2>&1; echo "rc=$?" >> gpurun_out/ab3/t_hq.log
python bench.py --n 1024 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab3/plain.json 2>&1
ARENA_FFT_QUAD=hq python bench.py --n 1024 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab3/hq_jr2.json 2>&1
for v in jr1 jr4; do
ARENA_FFT_QUAD=hq ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib python bench.py --n 1024 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab3/hq_$v.json 2>&1
done
python tools/ab_summary.py gpurun_out/ab3/*.json > gpurun_out/ab3/summary.txt 2>&1
