#!/bin/bash
# ncu --set full of the five kernels of one solve, plain and i-split (hq); summaries written on the box
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
for mode in plain hq; do
  env_q=""; [ $mode = hq ] && env_q="ARENA_FFT_QUAD=hq"
  env $env_q timeout 900 ncu --set full --clock-control none --import-source on -c 5 -o /tmp/ncu_$mode -f python tools/solve_once.py --reps 1 > gpurun_out/ncu/ncu_$mode.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$mode.ncu-rep > gpurun_out/ncu/summary_$mode.txt 2>&1
  for k in k_strided_tma k_zfwd k_zinv; do
    python tools/ncu_stalls.py /tmp/ncu_$mode.ncu-rep "$k" 30 > gpurun_out/ncu/stalls_${mode}_$k.txt 2>&1
  done
done
ls -la /tmp/ncu_*.ncu-rep >> gpurun_out/ncu/ncu_plain.log
