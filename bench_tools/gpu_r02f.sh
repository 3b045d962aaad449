# r02f: bwd main Q/dO L2 prefetch A/B (0 / 2 / 3 items ahead) + trace with prefetch
T=r02f
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=nopf EXTRA=-DTTT_BWD_PREFETCH=0 >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=pf3 EXTRA=-DTTT_BWD_PREFETCH=3 >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=trace EXTRA=-DTTT_TRACE >> gpurun_out/${T}_build.txt 2>&1
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_nopf.so build/libtttattn_pf3.so 2>&1 | tee gpurun_out/${T}_ab.txt
TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_bwd.py 40 timeline > gpurun_out/${T}_trace_timeline.txt 2>&1
grep -A22 "items " gpurun_out/${T}_trace_timeline.txt | head -22
timeout 600 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py -m gpu -q -x 2>&1 | tail -3
