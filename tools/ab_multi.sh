#!/bin/bash
# A/B of variants/*/lib over several bench configurations: tools/ab_multi.sh "args1" "args2" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
i=0
for cfg in "$@"; do
  i=$((i+1))
  python bench.py $cfg --no-cpu --no-e2e > gpurun_out/ab/base_c$i.json 2>&1
  for d in variants/*/; do v=$(basename $d); ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib python bench.py $cfg --no-cpu --no-e2e > gpurun_out/ab/${v}_c$i.json 2>&1; done
  echo "== $cfg"; python tools/ab_summary.py gpurun_out/ab/*_c$i.json
done
