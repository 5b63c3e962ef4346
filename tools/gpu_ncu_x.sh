#!/bin/bash
# ncu --set full + source-level stall samples (by opcode) of the x pass of one 1024^3 fp64 solve
cd "$(dirname "$0")/.."
O=gpurun_out/ncux; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_strided_tma --launch-skip 1 --launch-count 1 -o /tmp/ncu_x -f python tools/solve_once.py --reps 1 > $O/ncu_x.log 2>&1
python tools/ncu_summary.py /tmp/ncu_x.ncu-rep > $O/summary_x.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_x.ncu-rep k_strided_tma 40 > $O/stalls_x.txt 2>&1
