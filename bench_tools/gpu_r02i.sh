T=r02i
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so 2>&1 | tee gpurun_out/${T}_ab.txt
timeout 900 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py -m gpu -q -x 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ttt_bwd_pre -c 1 -o gpurun_out/${T}_pre_unroll python bench_tools/prof_unroll.py > gpurun_out/${T}_ncu1.log 2>&1
