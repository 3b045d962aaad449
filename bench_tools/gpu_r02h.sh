T=r02h
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=ord1 EXTRA=-DTTT_BWD_ORDER=1 >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=dqred EXTRA=-DTTT_BWD_DQ_RED=1 >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=both EXTRA="-DTTT_BWD_DQ_RED=1 -DTTT_BWD_ORDER=1" >> gpurun_out/${T}_build.txt 2>&1
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_ord1.so build/libtttattn_dqred.so build/libtttattn_both.so 2>&1 | tee gpurun_out/${T}_ab.txt
for v in ord1 dqred; do TTT_ATTN_LIB=build/libtttattn_$v.so timeout 300 python -m pytest tests/test_gpu_bwd_bf16.py -m gpu -q -x 2>&1 | tail -2; done
