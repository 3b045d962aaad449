#!/bin/bash
# A/B(/C...) kernel timing in one GPU session: bench_tools/ab.sh rounds lib1.so lib2.so [...]
# alternates time_kernels.py runs so clock / box drift affects all sides equally
R=$1; shift
for r in $(seq $R); do
  for v in "$@"; do
    echo "== $v"; TTT_ATTN_LIB=$v timeout 300 python bench_tools/time_kernels.py llama8b bwd 2>&1 | tail -2
  done
done
