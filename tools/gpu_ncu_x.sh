#!/bin/bash
# ncu --set full + source-level stall samples of the x pass: default kernel and the two-group kernel
cd "$(dirname "$0")/.."
O=gpurun_out/ncux; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_strided_tma --launch-skip 1 --launch-count 1 -o /tmp/ncu_x -f python tools/solve_once.py --reps 1 > $O/ncu_x.log 2>&1
python tools/ncu_summary.py /tmp/ncu_x.ncu-rep > $O/summary_x.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_x.ncu-rep k_strided_tma 60 > $O/stalls_x.txt 2>&1
ARENA_FFT_XPP=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_xpass_pp --launch-count 1 -o /tmp/ncu_xpp -f python tools/solve_once.py --reps 1 > $O/ncu_xpp.log 2>&1
python tools/ncu_summary.py /tmp/ncu_xpp.ncu-rep > $O/summary_xpp.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_xpp.ncu-rep k_xpass_pp 60 > $O/stalls_xpp.txt 2>&1
for k in x xpp; do
  ncu -i /tmp/ncu_$k.ncu-rep --page source --csv 2>/dev/null | gzip > $O/source_$k.csv.gz
  ncu -i /tmp/ncu_$k.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/raw_$k.csv.gz
done
ls -la $O
