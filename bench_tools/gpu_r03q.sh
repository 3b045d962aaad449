#!/bin/bash
# r03q: forward diagonal ring extended into the V stages for short CTAs (TTT_FWD_DG_EXT_NKV), no spills
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${T:-r03q}
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
for v in 0 2 8; do make variant VNAME=ext$v EXTRA="-DTTT_FWD_DG_EXT_NKV=$v" >> gpurun_out/${T}_build.txt 2>&1; done
make variant VNAME=wd EXTRA="-DTTT_WATCHDOG" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py -m gpu -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_packed.py tests/test_gpu_tree.py tests/test_gpu_bwd_bf16.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/${T}_pytest.txt

bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_ext0.so build/libtttattn_ext2.so build/libtttattn_ext8.so build/libtttattn_prev.so 2>&1 | tee gpurun_out/${T}_ab.txt
for v in ext0 ext8; do TTT_ATTN_LIB=build/libtttattn_$v.so python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"; done
python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ext4', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"
