#!/bin/bash
# r04e: forward diagonal math factored into shared device functions (diagonal warps + short-CTA helpers):
# parity and an A/B against the previous HEAD (build/prev_csrc)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r04e
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=shd16 EXTRA="-DTTT_FWD_SHD_NKV=16" >> gpurun_out/${T}_build.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_packed.py tests/test_gpu_edge_cases.py tests/test_gpu_autograd.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/${T}_pytest.txt
TTT_ATTN_LIB=build/libtttattn_shd16.so timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_packed.py -m gpu -q -x 2>&1 | tail -2
bash bench_tools/ab_lib.sh $T 3 paper_2603_18567_b200/libtttattn.so build/libtttattn_prev.so 2>&1 | tee gpurun_out/${T}_ab.txt
