#!/bin/bash
# r03k: dq = bf16(dq_acc) fused into the bwd main kernel (TTT_BWD_FCVT: per-tile counters, q-tile-major items)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03k
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=nofcvt EXTRA="-DTTT_BWD_FCVT=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA="-DTTT_WATCHDOG" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_bwd_bf16.py -m gpu -q -x -k "small or tiny or determin" 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_packed.py tests/test_gpu_autograd.py tests/test_gpu_head_parallel.py tests/test_gpu_draft.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 3 paper_2603_18567_b200/libtttattn.so build/libtttattn_nofcvt.so 2>&1 | tee gpurun_out/${T}_ab.txt
