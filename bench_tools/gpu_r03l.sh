#!/bin/bash
# r03l: bwd item order q-tile-major descending (TTT_BWD_QT_MAJOR) without the fused convert; FCVT=1 packed test
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03l
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=qtm EXTRA="-DTTT_BWD_QT_MAJOR=1" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_qtm.so timeout 900 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_packed.py -m gpu -q -x 2>&1 | tail -3
bash bench_tools/ab_lib.sh $T 3 paper_2603_18567_b200/libtttattn.so build/libtttattn_qtm.so 2>&1 | tee gpurun_out/${T}_ab.txt
