#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/tr
python -m pytest tests/test_parity_gpu.py tests/test_headline_gpu.py -m gpu -x -q -k "golden or random or config or pencil or quadrant or split3 or headline or 1024" > gpurun_out/tr/t.log 2>&1; echo "rc=$?" >> gpurun_out/tr/t.log
for r in 1 2; do
python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/tr/tw1_$r.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/twrec0/lib python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/tr/tw0_$r.json 2>&1
done
for r in 1; do
python bench.py --precision 32 --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/tr/tw1_f32_$r.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/twrec0/lib python bench.py --precision 32 --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/tr/tw0_f32_$r.json 2>&1
done
python tools/ab_summary.py gpurun_out/tr/*.json > gpurun_out/tr/summary.txt 2>&1
