T=r02g
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=trace EXTRA=-DTTT_TRACE >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_bwd.py 40 timeline > gpurun_out/${T}_trace_timeline.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_bwd.py 300 timeline > gpurun_out/${T}_trace_timeline300.txt 2>&1
grep -B2 -A80 "P arrive" gpurun_out/${T}_trace_timeline.txt | tail -75
