#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/xw
for r in 1 2; do
python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/xw/base_$r.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/xw0/lib python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/xw/xw0_$r.json 2>&1
done
python tools/ab_summary.py gpurun_out/xw/*.json > gpurun_out/xw/summary.txt 2>&1
