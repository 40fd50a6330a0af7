#!/bin/bash
# A/B of the bucket join's carried payload (scripts/join_probe.py, 1e8 rows a side)
for m in carry nocarry; do
  if [ $m = nocarry ]; then export RL_BJ_NO_CARRY=1; else unset RL_BJ_NO_CARRY; fi
  echo "== $m"; python scripts/join_probe.py ${1:-1e8} 4 bucket | tail -2
done
