# forward pipeline traces: per-CTA start -> first S, tile period, last S -> end (j = 0 and j = 6)
T=r02j
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=trace EXTRA=-DTTT_TRACE >> gpurun_out/${T}_build.txt 2>&1
for j in 0 6; do for c in 0 5 600 1200 1700 2040; do
  TTT_TRACE_STEP=$j TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_fwd.py $c > gpurun_out/${T}_ftrace_j${j}_c${c}.txt 2>&1
  echo "j=$j $(tail -1 gpurun_out/${T}_ftrace_j${j}_c${c}.txt)"
done; done
