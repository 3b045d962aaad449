#!/bin/bash
# r04g: forward diagonal steps as extra tensor-core kv tiles with a diagonal-only mask (TTT_FWD_TC_DIAG=1)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${T:-r04g}
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=tcd EXTRA="-DTTT_FWD_TC_DIAG=1" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=tcdwd EXTRA="-DTTT_FWD_TC_DIAG=1 -DTTT_WATCHDOG" >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_tcdwd.so timeout 300 python -m pytest tests/test_gpu_fwd_bf16.py -m gpu -q -x -k small 2>&1 | tail -3
TTT_ATTN_LIB=build/libtttattn_tcd.so timeout 1500 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_ttt_length.py tests/test_gpu_packed.py tests/test_gpu_edge_cases.py tests/test_gpu_bwd_bf16.py tests/test_gpu_autograd.py tests/test_gpu_dp_shard.py -m gpu -q -x 2>&1 | tail -4 | tee gpurun_out/${T}_pytest.txt
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_tcd.so 2>&1 | tee gpurun_out/${T}_ab.txt
TTT_ATTN_LIB=build/libtttattn_tcd.so python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tcd', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"
python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"
