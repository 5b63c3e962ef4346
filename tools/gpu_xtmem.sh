#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/xt2
python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/xt2/base.json 2>&1
ARENA_FFT_XTMEM=1 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/xt2/xtmem_pf1.json 2>&1
ARENA_FFT_XTMEM=1 ARENA_FFT_LIB_DIR=$PWD/variants/xtpf0/lib python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/xt2/xtmem_pf0.json 2>&1
python tools/ab_summary.py gpurun_out/xt2/*.json > gpurun_out/xt2/summary.txt 2>&1
ARENA_FFT_XTMEM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_xpass_tmem -c 1 -o /tmp/ncu_xt -f python tools/solve_once.py --reps 1 > gpurun_out/xt2/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_xt.ncu-rep > gpurun_out/xt2/ncu_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_xt.ncu-rep k_xpass_tmem 40 > gpurun_out/xt2/ncu_stalls.txt 2>&1
