#!/bin/bash
# A/B of the two-group x pass (poisson_xpp.cuh, ARENA_FFT_XPP=1) against the default kernels, then parity.
cd "$(dirname "$0")/.."
O=gpurun_out/xpp; mkdir -p $O
B="--steps 20 --warmup 3 --no-cpu --no-e2e"
for r in 1 2; do
  python bench.py --n 1024 $B > $O/base_$r.json 2>&1
  ARENA_FFT_XPP=1 python bench.py --n 1024 $B > $O/xpp_$r.json 2>&1
  for d in variants/*/; do v=$(basename $d)
    ARENA_FFT_XPP=1 ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib python bench.py --n 1024 $B > $O/${v}_$r.json 2>&1
  done
done
python bench.py --n 1024 --precision 32 $B > $O/base32.json 2>&1
ARENA_FFT_XPP=1 python bench.py --n 1024 --precision 32 $B > $O/xpp32.json 2>&1
python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > $O/base_2048.json 2>&1
ARENA_FFT_XPP=1 python bench.py --n 2048 --steps 5 --warmup 2 --no-cpu --no-e2e > $O/xpp_2048.json 2>&1
python tools/ab_summary.py $O/*.json > $O/summary.txt 2>&1
ARENA_FFT_XPP=1 timeout 900 python -m pytest tests/test_headline_gpu.py -m gpu -x -q -k "device_vs_oracle or fp32" > $O/t_headline.log 2>&1; echo "rc=$?" >> $O/t_headline.log
cat $O/summary.txt; tail -n 3 $O/t_headline.log
