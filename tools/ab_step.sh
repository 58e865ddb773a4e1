#!/bin/bash
# A/B timing of two builds of the library on the same box: alternates processes
# A B A B ... running tools/probe_step.py and prints the per-step times of the last steps.
# usage: tools/ab_step.sh abtest/libA.so abtest/libB.so [model] [batch] [rounds]
A=$1; B=$2; M=${3:-vgg16}; BS=${4:-128}; R=${5:-3}
for r in $(seq 1 $R); do
  for L in $A $B; do
    echo "== $L"
    RALPB_LIB=$L python tools/probe_step.py $M $BS 2>&1 | tail -3 | awk '{print $4, $5, $6, $7, $8, $9, $10, $11, $12, $13}'
  done
done
