#!/bin/bash
# A/B builds: usage: build_variant.sh <radix_sort.cu variant> <out.so> (the other objects from csrc/build).
# Put <out.so> inside the repo (it must travel with gpurun) and select it with RELAB_B200_LIB=<out.so>.
set -e
C=/root/repo/paper_2602_21237_b200/csrc
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Xcompiler -pthread -I$C -c "$1" -o /tmp/rs_variant.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$2" /tmp/rs_variant.o $(ls $C/build/*.o | grep -v radix_sort) -cudart static -Xcompiler -pthread
