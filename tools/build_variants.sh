#!/bin/bash
# Build kernel-tuning variants side by side: variants/<name>/lib/libarena_fft.so
# usage: tools/build_variants.sh name1="-DFLAG=.. -DFLAG2=.." name2="..."
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
for spec in "$@"; do
  name="${spec%%=*}"; flags="${spec#*=}"
  make -s -C paper_1408_6497_b200 -j8 OBJ=$PWD/variants/$name/build LIB=$PWD/variants/$name/lib \
       EXTRA_NVFLAGS="$flags" > variants/$name.buildlog 2>&1 || { echo "build $name failed"; tail variants/$name.buildlog; exit 1; } &
done
wait
ls variants/*/lib/libarena_fft.so
