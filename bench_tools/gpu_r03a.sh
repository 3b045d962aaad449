#!/bin/bash
# r03a: TMEM read/write bandwidth microbenchmark; forward softmax one-read (TTT_FWD_ONEREAD) and bwd dQ
# drain in halves (TTT_BWD_DQ_HALVES): watchdog smoke, parity tests, interleaved A/B vs the previous form
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03a
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=base EXTRA="-DTTT_FWD_ONEREAD=0 -DTTT_BWD_DQ_HALVES=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=fwdonly EXTRA="-DTTT_BWD_DQ_HALVES=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA=-DTTT_WATCHDOG >> gpurun_out/${T}_build.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/tmem_bw bench_tools/tmem_bw.cu > /dev/null 2>&1
timeout 120 ./build/tmem_bw > gpurun_out/${T}_tmem_bw.txt 2>&1; cat gpurun_out/${T}_tmem_bw.txt
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_bwd_bf16.py -m gpu -q -x -k "small or tiny or determin" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_bwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_tree.py tests/test_gpu_packed.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 3 paper_2603_18567_b200/libtttattn.so build/libtttattn_base.so build/libtttattn_fwdonly.so 2>&1 | tee gpurun_out/${T}_ab.txt
