#!/bin/bash
# A/B of the two-group x pass (poisson_xpp.cuh, ARENA_FFT_XPP=1) against the default kernels.
cd "$(dirname "$0")/.."
O=gpurun_out/xpp2; mkdir -p $O
B="--steps 20 --warmup 3 --no-cpu --no-e2e"
for r in 1 2; do
  timeout 200 python bench.py --n 1024 $B > $O/base_$r.json 2>&1
  ARENA_FFT_XPP=1 timeout 200 python bench.py --n 1024 $B > $O/xpp_skew1_$r.json 2>&1
  for d in variants/*/; do v=$(basename $d)
    ARENA_FFT_XPP=1 ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib timeout 200 python bench.py --n 1024 $B > $O/xpp_${v}_$r.json 2>&1
  done
done
python tools/ab_summary.py $O/*.json
