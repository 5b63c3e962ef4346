#!/bin/bash
# A/B of the shifted last exchange (E2S) in the strided passes, then the GPU parity suite.
cd "$(dirname "$0")/.."
O=gpurun_out/e2s; mkdir -p $O
B="--steps 20 --warmup 3 --no-cpu --no-e2e"
for r in 1 2; do
  timeout 300 python bench.py --n 1024 $B > $O/e2s_$r.json 2>&1
  for d in variants/*/; do v=$(basename $d)
    ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib timeout 300 python bench.py --n 1024 $B > $O/${v}_$r.json 2>&1
  done
done
timeout 300 python bench.py --n 1024 --precision 32 $B > $O/e2s_32.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/e2s0/lib timeout 300 python bench.py --n 1024 --precision 32 $B > $O/e2s0_32.json 2>&1
timeout 300 python bench.py --n 512 $B > $O/e2s_512.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/e2s0/lib timeout 300 python bench.py --n 512 $B > $O/e2s0_512.json 2>&1
timeout 300 python bench.py --n 256 $B > $O/e2s_256.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/e2s0/lib timeout 300 python bench.py --n 256 $B > $O/e2s0_256.json 2>&1
timeout 400 python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > $O/e2s_2048.json 2>&1
ARENA_FFT_LIB_DIR=$PWD/variants/e2s0/lib timeout 400 python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > $O/e2s0_2048.json 2>&1
python tools/ab_summary.py $O/*.json > $O/summary.txt 2>&1
cat $O/summary.txt
timeout 2400 python -m pytest tests -m gpu -x -q > $O/t_gpu.log 2>&1; echo "rc=$?" >> $O/t_gpu.log
tail -n 5 $O/t_gpu.log
