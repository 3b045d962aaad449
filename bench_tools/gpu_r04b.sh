#!/bin/bash
# r04b: bwd dS phase with one 64-column dP^T load (TTT_BWD_DS_ONEWAIT, compute warps 152 registers)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r04b
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=ow0 EXTRA="-DTTT_BWD_DS_ONEWAIT=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=ow0r152 EXTRA="-DTTT_BWD_DS_ONEWAIT=0 -DTTT_BWD_REG_CMP=152" >> gpurun_out/${T}_build.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py tests/test_gpu_packed.py tests/test_gpu_edge_cases.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 3 paper_2603_18567_b200/libtttattn.so build/libtttattn_ow0.so build/libtttattn_ow0r152.so 2>&1 | tee gpurun_out/${T}_ab.txt
