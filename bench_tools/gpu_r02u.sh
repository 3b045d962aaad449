T=r02u
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA=-DTTT_WATCHDOG >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=dnomath EXTRA=-DTTT_FWD_DIAG_MODE=1 >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_fwd_bf16.py -m gpu -q -x -k "small or determin" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_tree.py tests/test_gpu_bwd_bf16.py -m gpu -q -x 2>&1 | tail -3
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_prev.so build/libtttattn_dnomath.so 2>&1 | tee gpurun_out/${T}_ab.txt
