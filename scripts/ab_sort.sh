#!/bin/bash
# A/B of the cfg2 bench step: the default library vs build_variants/$1.so, interleaved
for i in 1 2 3; do
  for lib in "" "build_variants/$1.so"; do
    RELAB_B200_LIB=$lib python bench.py --no-join --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${lib:-default}', d['ms_per_step'], d['roofline']['avg_launch_us'])"
  done
done
