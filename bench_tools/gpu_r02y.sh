#!/bin/bash
# r02y: PACKED as a template flag (padded instantiations unchanged): packed tests + A/B vs the pre-packed build
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
make -j8 > gpurun_out/r02y_build.txt 2>&1 || { tail -30 gpurun_out/r02y_build.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_check_mode.py tests/test_gpu_bwd_unroll.py -q > gpurun_out/r02y_packed.txt 2>&1; echo "rc=$?" >> gpurun_out/r02y_packed.txt
tail -4 gpurun_out/r02y_packed.txt
bash bench_tools/ab_lib.sh r02y 3 build/ab/lib_prepacked.so paper_2603_18567_b200/libtttattn.so
