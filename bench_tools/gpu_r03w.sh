#!/bin/bash
# r03w: this session's kernels (HEAD) vs the session-start build (0a32e6c, build/prev_csrc), interleaved
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03w
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
bash bench_tools/ab_lib.sh $T 4 paper_2603_18567_b200/libtttattn.so build/libtttattn_prev.so 2>&1 | tee gpurun_out/${T}_ab.txt
