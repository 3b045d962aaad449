T=r02t
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA=-DTTT_WATCHDOG >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=dkts EXTRA=-DTTT_BWD_DK_SS=0 >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_bwd_bf16.py -m gpu -q -x -k small 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py tests/test_gpu_fwd_bf16.py tests/test_gpu_edge_cases.py tests/test_gpu_ttt_length.py -m gpu -q -x 2>&1 | tail -2
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_dkts.so 2>&1 | tee gpurun_out/${T}_ab.txt
