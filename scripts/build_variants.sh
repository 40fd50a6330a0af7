#!/bin/bash
# Build librelab_b200 variants with different tuning macros into build_variants/.
# usage: scripts/build_variants.sh NAME "-DMACRO=1 ..." [NAME "-D..."]...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build_variants
mkdir -p $OUT
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  tmp=$(mktemp -d)
  for f in radix_sort key_axis expand capi stager digest plan exchange; do
    nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $defs -Xptxas -v \
      -c $ROOT/paper_2602_21237_b200/csrc/$f.cu -o $tmp/$f.o 2> $tmp/$f.log || { cat $tmp/$f.log; exit 1; }
  done
  grep -A2 onesweep $tmp/radix_sort.log | grep -E "Used|spill" | sed "s/^/[$name] /"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so $tmp/*.o -cudart static
  rm -rf $tmp
done
