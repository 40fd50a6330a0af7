#!/bin/bash
# A/B/... of the cfg2 bench step between library builds, interleaved: ab_libs.sh A.so B.so [C.so ...]
for i in 1 2 3; do
  for lib in "$@"; do
    RELAB_B200_LIB=$lib python bench.py --no-join --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$lib', d['ms_per_step'], r['avg_launch_us'], r['phases_last_step']['local_phase_us'])"
  done
done
