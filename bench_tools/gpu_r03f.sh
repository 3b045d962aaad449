#!/bin/bash
# r03f: bwd P phase: mask-free full-tile loop (TTT_BWD_PSPLIT), exp2 emulation fraction (TTT_BWD_EMU_MASK)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03f
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=nosplit EXTRA="-DTTT_BWD_PSPLIT=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=emu0 EXTRA="-DTTT_BWD_EMU_MASK=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=emu2 EXTRA="-DTTT_BWD_EMU_MASK=0xAA" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=emu8 EXTRA="-DTTT_BWD_EMU_MASK=0x80" >> gpurun_out/${T}_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_packed.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_nosplit.so build/libtttattn_emu0.so build/libtttattn_emu2.so build/libtttattn_emu8.so 2>&1 | tee gpurun_out/${T}_ab.txt
