#!/bin/bash
# Interleaved A/B of the bucket join (1e8 cfg5 shape, 1e8 cfg4 shape) between library builds: ab_join.sh A.so B.so ...
for i in 1 2; do
  for lib in "$@"; do
    a=$(RELAB_B200_LIB=$lib python scripts/join_probe.py 1e8 3 bucket | tail -1 | awk '{print $(NF-2)}')
    b=$(RELAB_B200_LIB=$lib PROBE_SHAPE=cfg4 python scripts/join_probe.py 1e8 3 bucket | tail -1 | awk '{print $(NF-2)}')
    echo "$lib cfg5-1e8 $a ms cfg4-1e8 $b ms"
  done
done
