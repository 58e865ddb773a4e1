#!/bin/bash
# A/B timing of two builds of the library on the same box: alternates processes
# A B A B ... running tools/probe_step.py and prints the median step time of steps 3..7
# of every process, then the per-build medians.
# usage: tools/ab_step.sh abtest/libA.so abtest/libB.so [model] [batch] [rounds]
A=$1; B=$2; M=${3:-vgg16}; BS=${4:-128}; R=${5:-3}
for r in $(seq 1 $R); do
  for L in $A $B; do
    RALPB_LIB_LENIENT=1 RALPB_LIB=$L python tools/probe_step.py $M $BS 2>&1 | awk -v L=$L '/^step [3-7]:/ {print L, $6, $8, $10, $12, $14}'
  done
done | python -c "
import sys, statistics, collections
d = collections.defaultdict(list)
for line in sys.stdin:
    p = line.split()
    d[p[0]].append([float(x.rstrip(')')) for x in p[1:]])
for k, v in d.items():
    cols = list(zip(*v))
    print(k, 'n=%d' % len(v), 'median ms %.3f (fwd %.3f back %.3f bwd %.3f sync %.3f)' % tuple(statistics.median(c) for c in cols),
          'min %.3f' % min(cols[0]))
"
