#!/bin/bash
# A/B of the split-exchange strided passes (HX) against the previous kernels, then parity.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/hx
for r in 1 2; do
  python bench.py --n 1024 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/hx/hx_$r.json 2>&1
  for v in hx0 hxy; do
    ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib python bench.py --n 1024 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/hx/${v}_$r.json 2>&1
  done
done
python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/hx/hx_2048.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/hx0/lib python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/hx/hx0_2048.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/hxy/lib python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/hx/hxy_2048.json 2>&1
python tools/ab_summary.py gpurun_out/hx/*.json > gpurun_out/hx/summary.txt 2>&1
timeout 900 python -m pytest tests/test_headline_gpu.py -m gpu -x -q -k "device_vs_oracle or fp32" > gpurun_out/hx/t_headline.log 2>&1; echo "rc=$?" >> gpurun_out/hx/t_headline.log
ARENA_FFT_LIB_DIR=$PWD/variants/hxy/lib timeout 900 python -m pytest tests/test_headline_gpu.py -m gpu -x -q -k "device_vs_oracle" > gpurun_out/hx/t_headline_hxy.log 2>&1; echo "rc=$?" >> gpurun_out/hx/t_headline_hxy.log
cat gpurun_out/hx/summary.txt; tail -3 gpurun_out/hx/t_headline.log gpurun_out/hx/t_headline_hxy.log
