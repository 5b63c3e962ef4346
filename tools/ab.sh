#!/bin/bash
# A/B timing of compile-time variants (variants/*/lib) on the GPU box: tools/ab.sh [n] [precision] [extra bench args]
n=${1:-1024}; prec=${2:-64}; extra=${3:-}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
timeout 300 python bench.py --n $n --precision $prec --steps 20 --warmup 3 --no-cpu --no-e2e $extra > gpurun_out/ab/base_${n}_${prec}.json 2>&1
for d in variants/*/; do
  v=$(basename $d)
  ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib timeout 300 python bench.py --n $n --precision $prec --steps 20 --warmup 3 --no-cpu --no-e2e $extra > gpurun_out/ab/${v}_${n}_${prec}.json 2>&1
done
python tools/ab_summary.py gpurun_out/ab/*_${n}_${prec}.json
