#!/bin/bash
# r03m: forward diagonal cost attribution after the one-read softmax: probes without the diagonal math (1) / loads (2)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03m
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
make variant VNAME=nomath EXTRA="-DTTT_FWD_DIAG_MODE=1" >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=noload EXTRA="-DTTT_FWD_DIAG_MODE=2" >> gpurun_out/${T}_build.txt 2>&1
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_nomath.so build/libtttattn_noload.so 2>&1 | tee gpurun_out/${T}_ab.txt
for v in nomath noload; do TTT_ATTN_LIB=build/libtttattn_$v.so python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"; done
python bench.py --no-e2e --no-cpu --no-loss --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])"
