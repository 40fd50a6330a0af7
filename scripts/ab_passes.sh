#!/bin/bash
# A/B of the counting passes: cfg2 sort step (bench, payload gathered / carried), cfg5 / cfg4 joins at 1e8, interleaved.
# usage: ab_passes.sh <variant.so> [rounds] [joins: 1|0]
for i in $(seq 1 ${2:-2}); do
  for lib in "$1" ""; do
    for carry in 0 1; do
      [ -n "$lib" ] && [ $carry = 1 ] && [ -z "$AB_CARRY_BOTH" ] && continue
      RL_SORT_CARRY=$carry RELAB_B200_LIB=$lib python bench.py --no-join --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('${lib:-new} carry=$carry step', d['ms_per_step'], 'sort_us', r['avg_launch_us'], [v for k,v in r['phases_last_step'].items() if k!='note'])"
    done
    if [ "${3:-1}" = 1 ]; then
      RELAB_B200_LIB=$lib python scripts/join_probe.py 1e8 4 bucket | tail -1
      PROBE_SHAPE=cfg4 RELAB_B200_LIB=$lib python scripts/join_probe.py 1e8 4 bucket | tail -1
    fi
  done
done
