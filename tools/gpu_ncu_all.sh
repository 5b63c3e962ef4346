#!/bin/bash
# ncu --set full of the five kernels of one 1024^3 fp64 solve; per-opcode stall tables written on the box
cd "$(dirname "$0")/.."
O=gpurun_out/ncuall; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -c 5 -o /tmp/ncu_all -f python tools/solve_once.py --reps 1 > $O/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_all.ncu-rep > $O/summary.txt 2>&1
i=0
for k in k_zfwd k_strided_tma k_zinv; do
  python tools/ncu_stalls.py /tmp/ncu_all.ncu-rep "$k" 40 > $O/stalls_$k.txt 2>&1
done
# the y kernels: first k_strided_tma launch is yfwd (ncu_stalls takes the first match)
ls -la $O
