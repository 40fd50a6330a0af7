#!/bin/bash
# A/B of the cfg2 bench step between two library builds, interleaved: ab_lib.sh A.so B.so
for i in 1 2 3; do
  for lib in "$1" "$2"; do
    RELAB_B200_LIB=$lib python bench.py --no-join --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', d['ms_per_step'], d['roofline']['avg_launch_us'], d['roofline']['phases_last_step'])"
  done
done
