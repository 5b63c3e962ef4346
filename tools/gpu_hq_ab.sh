#!/bin/bash
# i-split (hq) formulation: parity + A/B against the plain path at 1024^3 fp64/fp32
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "quadrant or repeat" > gpurun_out/t_hq.log 2>&1; echo "rc=$?" >> gpurun_out/t_hq.log
for prec in 64 32; do
  python bench.py --n 1024 --precision $prec --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/plain_$prec.json 2>&1
  ARENA_FFT_QUAD=hq python bench.py --n 1024 --precision $prec --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/hq_$prec.json 2>&1
  ARENA_FFT_QUAD=hq ARENA_FFT_LIB_DIR=$PWD/variants/xs16/lib python bench.py --n 1024 --precision $prec --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/hqxs16_$prec.json 2>&1
  ARENA_FFT_QUAD=1 ARENA_FFT_LIB_DIR=$PWD/variants/xs16/lib python bench.py --n 1024 --precision $prec --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/quadxs16_$prec.json 2>&1
done
python tools/ab_summary.py gpurun_out/ab/*.json > gpurun_out/ab/summary.txt 2>&1
