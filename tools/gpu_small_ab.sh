#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/small; mkdir -p $O
for n in 64 128 256 512; do for r in 1 2 3; do
  timeout 200 python bench.py --n $n --config 2 --steps 50 --warmup 10 --no-cpu --no-e2e > $O/base_${n}_$r.json 2>&1
  ARENA_FFT_LIB_DIR=$PWD/variants/e2s0/lib timeout 200 python bench.py --n $n --config 2 --steps 50 --warmup 10 --no-cpu --no-e2e > $O/e2s0_${n}_$r.json 2>&1
done; done
python tools/ab_summary.py $O/*.json
