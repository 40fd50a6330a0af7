for n in 1e6 2e6 4e6; do
  for sel in 0 1; do
    if [ $sel = 1 ]; then export RL_BJ_NO_SEL=1; else unset RL_BJ_NO_SEL; fi
    RL_FORCE_BJOIN=1 python scripts/join_probe.py $n 20 both 2>&1 | grep -E "join n=" | python -c "
import sys,collections,statistics
d=collections.defaultdict(list)
for l in sys.stdin:
    m=l.split(); d[m[0]].append(float(m[3]))
print('$n sel_off=$sel', {k: round(statistics.median(v),3) for k,v in d.items()})"
  done
done
