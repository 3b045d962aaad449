#!/bin/bash
# r03n: forward register split without spills (softmax 176, diagonal 120, role 40) vs the committed 168/128/48
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03n
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=r168 EXTRA="-DTTT_FWD_REG_SOFTMAX=168 -DTTT_FWD_REG_DIAG=128" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=r176d128 EXTRA="-DTTT_FWD_REG_SOFTMAX=176 -DTTT_FWD_REG_DIAG=128" >> gpurun_out/${T}_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_tree.py tests/test_gpu_packed.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 3 paper_2603_18567_b200/libtttattn.so build/libtttattn_r168.so build/libtttattn_r176d128.so 2>&1 | tee gpurun_out/${T}_ab.txt
