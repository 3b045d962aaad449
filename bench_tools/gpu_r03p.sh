#!/bin/bash
# r03p: Q / first K-V (fwd) and K / V / item 0 (bwd main) TMA loads issued with the barrier setup, before the
# TMEM allocation and the CTA barrier; A/B vs the previous HEAD (build/prev_csrc)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03p
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=wd EXTRA="-DTTT_WATCHDOG" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_bwd_bf16.py -m gpu -q -x -k "small or tiny or determin" 2>&1 | tail -2
timeout 1800 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_tree.py tests/test_gpu_packed.py tests/test_gpu_autograd.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 3 paper_2603_18567_b200/libtttattn.so build/libtttattn_prev.so 2>&1 | tee gpurun_out/${T}_ab.txt
