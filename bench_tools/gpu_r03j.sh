#!/bin/bash
# r03j: forward exp2 emulation fraction after the one-read softmax (TTT_FWD_EMU_MASK)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03j
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=e00 EXTRA="-DTTT_FWD_EMU_MASK=0x00" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=e80 EXTRA="-DTTT_FWD_EMU_MASK=0x80" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=eAA EXTRA="-DTTT_FWD_EMU_MASK=0xAA" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=eEE EXTRA="-DTTT_FWD_EMU_MASK=0xEE" >> gpurun_out/${T}_build.txt 2>&1
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_e00.so build/libtttattn_e80.so build/libtttattn_eAA.so build/libtttattn_eEE.so 2>&1 | tee gpurun_out/${T}_ab.txt
