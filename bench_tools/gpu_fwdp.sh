timeout 600 python -m pytest tests/test_gpu_fwd_bf16.py -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in paper_2603_18567_b200/libtttattn.so build/libtttattn_prev.so; do echo "== $v"; TTT_ATTN_LIB=$v timeout 200 python bench_tools/time_kernels.py llama8b | tail -1; done; done
