T=r02l
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=trace EXTRA=-DTTT_TRACE >> gpurun_out/${T}_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py -m gpu -q -x 2>&1 | tail -2
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so 2>&1 | tee gpurun_out/${T}_ab.txt
for j in 6; do for c in 0 600 2040; do
  TTT_TRACE_STEP=$j TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_fwd.py $c > gpurun_out/${T}_ftrace_j${j}_c${c}.txt 2>&1
  echo "j=$j $(tail -1 gpurun_out/${T}_ftrace_j${j}_c${c}.txt)"
done; done
