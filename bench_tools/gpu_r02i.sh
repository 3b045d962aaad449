T=r02i
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=pre7 EXTRA=-DTTT_PRE_WARPS=7 >> gpurun_out/${T}_build.txt 2>&1
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_pre7.so 2>&1 | tee gpurun_out/${T}_ab.txt
timeout 900 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py -m gpu -q -x 2>&1 | tail -3
TTT_ATTN_LIB=build/libtttattn_pre7.so timeout 900 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py -m gpu -q -x 2>&1 | tail -2
