#!/bin/bash
# Round-end measurement set on the GPU box (one gpurun call):
#   bench lines (fp64/fp32 1024^3, configs 1-3, 2048^3, reference arm), the ncu launch
#   list of the default bench command, and one ncu --set full capture of a solve
#   (summarised on the box: the report itself exceeds gpurun's 64 MiB return limit).
# Outputs under gpurun_out/prof/ (copied into profiles/ by hand after review).
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/prof
mkdir -p $O
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_1024_fp64.json 2> $O/bench_1024_fp64.err; echo "bench fp64 rc=$?"
timeout 1500 python bench.py --precision 32 --no-cpu > $O/bench_1024_fp32.json 2> $O/bench_1024_fp32.err; echo "bench fp32 rc=$?"
timeout 1500 python bench.py --n 512 --config 3 --no-cpu > $O/bench_512_fp64_config3.json 2>&1; echo "bench 512 rc=$?"
timeout 1500 python bench.py --n 256 --config 2 --no-cpu > $O/bench_256_fp64_config2.json 2>&1; echo "bench 256 rc=$?"
timeout 1500 python bench.py --n 64 --config 1 --no-cpu > $O/bench_64_fp64_config1.json 2>&1; echo "bench 64 rc=$?"
timeout 1500 python bench.py --n 2048 --config 5 --steps 5 --no-cpu > $O/bench_2048_fp64_config5.json 2>&1; echo "bench 2048 rc=$?"
timeout 1500 python bench.py --n 2048 --config 5 --precision 32 --steps 5 --no-cpu > $O/bench_2048_fp32_config5.json 2>&1; echo "bench 2048 fp32 rc=$?"
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err; echo "reference rc=$?"
timeout 1500 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/bench_small.json 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_1024_fp64.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/solve_once.py --n 1024 --reps 1 > $O/solve_once.log 2>&1 && \
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_z|k_strided" -c 5 -o /tmp/full_1024_fp64 -f \
      python tools/solve_once.py --n 1024 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/full_1024_fp64.ncu-rep --traffic 1024_64 > $O/ncu_full_summary.txt 2>&1
cp profiles/traffic_latest.json $O/traffic_latest.json
python tools/ncu_stalls.py /tmp/full_1024_fp64.ncu-rep "k_strided_tma<double, 1024, 2" 40 > $O/ncu_x_stalls.txt 2>&1
