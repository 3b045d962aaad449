#!/bin/bash
# r03d: Q / dO / lse2 / Delta loads of the bwd main kernel by cp.async (LSU path, TTT_BWD_LSU_LOADS) instead of
# TMA; A/B: {DQT 1, 0} x {LSU 1, 0}; traces of the LSU variants
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03d
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=lsu0 EXTRA="-DTTT_BWD_DQT=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=prev EXTRA="-DTTT_BWD_DQT=0 -DTTT_BWD_LSU_LOADS=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA="-DTTT_WATCHDOG" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd0 EXTRA="-DTTT_WATCHDOG -DTTT_BWD_DQT=0" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_bwd_bf16.py -m gpu -q -x -k "small or tiny or determin" 2>&1 | tail -2
TTT_ATTN_LIB=build/libtttattn_wd0.so timeout 300 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_packed.py -m gpu -q -x 2>&1 | tail -2
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_lsu0.so build/libtttattn_prev.so 2>&1 | tee gpurun_out/${T}_ab.txt
make variant VNAME=tr1 EXTRA="-DTTT_TRACE" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=tr0 EXTRA="-DTTT_TRACE -DTTT_BWD_DQT=0" >> gpurun_out/${T}_build.txt 2>&1
for v in tr0 tr1; do
  TTT_ATTN_LIB=build/libtttattn_$v.so timeout 120 python bench_tools/trace_bwd.py 40 timeline > gpurun_out/${T}_${v}_timeline.txt 2>&1
  grep -A24 "period" gpurun_out/${T}_${v}_timeline.txt | head -25
done
timeout 1500 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_packed.py tests/test_gpu_autograd.py tests/test_gpu_check_mode.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/${T}_pytest.txt
