timeout 600 python -m pytest tests/test_gpu_loss.py -x -q 2>&1 | tail -2 > gpurun_out/ab5_pytest.txt
for r in 1 2; do for v in paper_2603_18567_b200/libtttattn.so build/libtttattn_t1024.so build/libtttattn_t256.so; do TTT_ATTN_LIB=$v timeout 120 python bench_tools/time_loss.py; done; done > gpurun_out/ab5_loss.txt 2>&1
cat gpurun_out/ab5_pytest.txt gpurun_out/ab5_loss.txt
