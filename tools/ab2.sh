#!/bin/bash
# Environment-switch A/B on the GPU box: TMA strided kernels vs classic.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
n=${1:-1024}; prec=${2:-64}
python bench.py --n $n --precision $prec --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/tma_${n}_${prec}.json 2>&1
ARENA_FFT_KERNELS=classic python bench.py --n $n --precision $prec --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/classic_${n}_${prec}.json 2>&1
python tools/ab_summary.py gpurun_out/ab/tma_${n}_${prec}.json gpurun_out/ab/classic_${n}_${prec}.json
