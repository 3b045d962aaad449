#!/bin/bash
# r03g: forward CTA traces after the one-read softmax (long CTA 0 / short CTA 2040, j = 0 and 6)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03g
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || exit 1
make variant VNAME=trace EXTRA=-DTTT_TRACE >> gpurun_out/${T}_build.txt 2>&1
for j in 0 6; do for c in 0 2040; do
TTT_TRACE_STEP=$j TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_fwd.py $c > gpurun_out/${T}_ftrace_j${j}_c${c}.txt 2>&1
done; done
head -60 gpurun_out/${T}_ftrace_j0_c0.txt; tail -30 gpurun_out/${T}_ftrace_j0_c0.txt
head -50 gpurun_out/${T}_ftrace_j6_c2040.txt
