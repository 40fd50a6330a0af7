#!/bin/bash
# Interleaved A/B of the bucket join between library builds: ab_bj_libs.sh N A.so B.so ...
N=$1; shift
for i in 1 2; do
  for lib in "$@"; do
    echo "$lib $(RELAB_B200_LIB=$lib python scripts/join_probe.py $N 3 bucket | tail -1)"
  done
done
