#!/bin/bash
# Interleaved A/B of the 1e9 bucket join between library builds: ab_join1e9.sh A.so B.so ...
for i in 1 2; do
  for lib in "$@"; do
    echo "$lib $(RELAB_B200_LIB=$lib python scripts/join_probe.py 1e9 2 bucket | tail -1)"
  done
done
