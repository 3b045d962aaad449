#!/bin/bash
# r03e: bwd main timing probes: no dQ reduce-adds (PROBE=1), no Q/dO loads after item 1 (PROBE=2)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03e
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=p1 EXTRA="-DTTT_BWD_PROBE=1" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=p2 EXTRA="-DTTT_BWD_PROBE=2" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=p3 EXTRA="-DTTT_BWD_PROBE=1 -DTTT_BWD_DQT=1" >> gpurun_out/${T}_build.txt 2>&1
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_p1.so build/libtttattn_p2.so build/libtttattn_p3.so 2>&1 | tee gpurun_out/${T}_ab.txt
