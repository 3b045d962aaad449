T=r02m
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=trace EXTRA=-DTTT_TRACE >> gpurun_out/${T}_build.txt 2>&1
TTT_TRACE_STEP=6 TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_fwd.py 2040 > gpurun_out/${T}_ftrace_j6_c2040.txt 2>&1
grep -v "^ *[0-9]* *dgp" gpurun_out/${T}_ftrace_j6_c2040.txt | head -80
timeout 900 python -m pytest tests/test_gpu_draft.py -m gpu -q -x 2>&1 | tail -4
