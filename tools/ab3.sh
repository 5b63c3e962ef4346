#!/bin/bash
# Env-switch A/B: fused vs unfused z+y, lag values.  tools/ab3.sh [n] [prec]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
n=${1:-1024}; prec=${2:-64}
for cfg in "fused:" "unfused:ARENA_FFT_FUSED=0" "lag1:ARENA_FFT_FUSED_LAG=1" "lag4:ARENA_FFT_FUSED_LAG=4" "lag8:ARENA_FFT_FUSED_LAG=8"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs python bench.py --n $n --precision $prec --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab/${name}_${n}_${prec}.json 2>&1
done
python tools/ab_summary.py gpurun_out/ab/{fused,unfused,lag1,lag4,lag8}_${n}_${prec}.json
