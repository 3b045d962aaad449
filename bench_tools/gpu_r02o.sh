# persistent forward: watchdog-build smoke first (a deadlock traps instead of hanging), then tests and A/B
T=r02o
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA=-DTTT_WATCHDOG >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 180 python -m pytest tests/test_gpu_fwd_bf16.py -m gpu -q -x -k "small or determin" 2>&1 | tail -3
rc=$?
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 120 python bench_tools/prof_one.py llama8b 6 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_tree.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_bwd_bf16.py -m gpu -q -x 2>&1 | tail -3
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_prev.so 2>&1 | tee gpurun_out/${T}_ab.txt
