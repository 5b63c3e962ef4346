#!/bin/bash
# A/B of the FMA-form radix-4 DFT step (ARENA_DFT_FMA) against the previous engine, then the GPU parity suite.
cd "$(dirname "$0")/.."
O=gpurun_out/fma32; mkdir -p $O
B="--steps 20 --warmup 3 --no-cpu --no-e2e"
for r in 1 2 3; do
  timeout 300 python bench.py --n 1024 $B > $O/fma32_$r.json 2>&1
  for d in variants/*/; do v=$(basename $d)
    ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib timeout 300 python bench.py --n 1024 $B > $O/${v}_$r.json 2>&1
  done
done
for n in 512 256; do
timeout 300 python bench.py --n $n $B > $O/fma32_$n.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/e2sx/lib timeout 300 python bench.py --n $n $B > $O/e2sx_$n.json 2>&1
done
timeout 400 python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > $O/fma32_2048.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/e2sx/lib timeout 400 python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > $O/e2sx_2048.json 2>&1
python tools/ab_summary.py $O/*.json > $O/summary.txt 2>&1
cat $O/summary.txt
timeout 2400 python -m pytest tests -m gpu -x -q > $O/t_gpu.log 2>&1; echo "rc=$?" >> $O/t_gpu.log
tail -n 5 $O/t_gpu.log
