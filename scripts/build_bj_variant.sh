#!/bin/bash
# A/B builds of the bucket join: usage: build_bj_variant.sh <bucket_join.cu variant> <out.so> [extra nvcc flags]
# (the other objects from csrc/build); select the result with RELAB_B200_LIB=<out.so>.
set -e
C=/root/repo/paper_2602_21237_b200/csrc
SRC="$1"; OUT="$2"; shift 2
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Xcompiler -pthread -I$C "$@" -c "$SRC" -o /tmp/bj_variant_$$.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" /tmp/bj_variant_$$.o $(ls $C/build/*.o | grep -v bucket_join) -cudart static -Xcompiler -pthread
