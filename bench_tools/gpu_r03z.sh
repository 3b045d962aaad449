#!/bin/bash
# r03z: short-CTA diagonal on the softmax warps (TTT_FWD_SHD_NKV): parity (default and forced everywhere), A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03z
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
for v in 0 2 8 16; do make variant VNAME=shd$v EXTRA="-DTTT_FWD_SHD_NKV=$v" >> gpurun_out/${T}_build.txt 2>&1; done
make variant VNAME=wd EXTRA="-DTTT_WATCHDOG -DTTT_FWD_SHD_NKV=16" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 300 python -m pytest tests/test_gpu_fwd_bf16.py -m gpu -q -x -k "small" 2>&1 | tail -2
TTT_ATTN_LIB=build/libtttattn_shd16.so timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_packed.py tests/test_gpu_edge_cases.py -m gpu -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_packed.py tests/test_gpu_tree.py tests/test_gpu_autograd.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_shd0.so build/libtttattn_shd2.so build/libtttattn_shd8.so 2>&1 | tee gpurun_out/${T}_ab.txt
for v in shd0 shd8; do TTT_ATTN_LIB=build/libtttattn_$v.so python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"; done
python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('shd4', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"
