#!/bin/bash
# A/B timing of kernel variants on the GPU box: tools/ab.sh [n] [precision] [extra env for all runs]
n=${1:-1024}; prec=${2:-64}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
python bench.py --n $n --precision $prec --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/base_${n}_${prec}.json 2>&1
ARENA_FFT_KERNELS=classic python bench.py --n $n --precision $prec --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/baseclassic_${n}_${prec}.json 2>&1
for d in variants/*/; do
  v=$(basename $d)
  for mode in tma classic; do
    ARENA_FFT_KERNELS=$mode ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib python bench.py --n $n --precision $prec --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/${v}${mode}_${n}_${prec}.json 2>&1
  done
done
python tools/ab_summary.py gpurun_out/ab/*_${n}_${prec}.json
