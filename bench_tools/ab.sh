#!/bin/bash
# A/B kernel timing in one GPU session: bench_tools/ab.sh libA.so libB.so [rounds]
# alternates time_kernels.py runs so clock / box drift affects both sides equally
A=$1; B=$2; R=${3:-2}
for r in $(seq $R); do
  for v in $A $B; do
    echo "== $v"; TTT_ATTN_LIB=$v timeout 300 python bench_tools/time_kernels.py llama8b bwd 2>&1 | tail -2
  done
done
