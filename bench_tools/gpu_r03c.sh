#!/bin/bash
# r03c: bwd CTA pipeline traces, per-tile dQ (DQT=0) vs per-sub-item dQ^T (DQT=1)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03c
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=tr1 EXTRA="-DTTT_TRACE" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=tr0 EXTRA="-DTTT_TRACE -DTTT_BWD_DQT=0" >> gpurun_out/${T}_build.txt 2>&1
for v in tr0 tr1; do
  TTT_ATTN_LIB=build/libtttattn_$v.so timeout 120 python bench_tools/trace_bwd.py 40 timeline > gpurun_out/${T}_${v}_timeline.txt 2>&1
done
grep -A30 "period" gpurun_out/${T}_tr0_timeline.txt | head -32
grep -A30 "period" gpurun_out/${T}_tr1_timeline.txt | head -32
