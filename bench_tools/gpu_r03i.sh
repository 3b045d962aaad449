#!/bin/bash
# r03i: forward diagonal ring extended into the K stages for short CTAs (TTT_FWD_DG_EXT_NKV), out_lo staged in V
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03i
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=ext0 EXTRA="-DTTT_FWD_DG_EXT_NKV=0" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=ext2 EXTRA="-DTTT_FWD_DG_EXT_NKV=2" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=ext6 EXTRA="-DTTT_FWD_DG_EXT_NKV=6" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA="-DTTT_WATCHDOG" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_fwd_bf16.py -m gpu -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_tree.py tests/test_gpu_packed.py tests/test_gpu_autograd.py tests/test_gpu_bwd_bf16.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_ext0.so build/libtttattn_ext2.so build/libtttattn_ext6.so 2>&1 | tee gpurun_out/${T}_ab.txt
python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['per_ttt_step_ms'])"
TTT_ATTN_LIB=build/libtttattn_ext0.so python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['per_ttt_step_ms'])"
