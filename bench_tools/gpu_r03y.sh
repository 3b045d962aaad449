#!/bin/bash
# r03y: forward CTA order batch sweep (the model picks 32 groups at the Llama shape)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03y
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
bash bench_tools/ab_env.sh $T 3 "-" "TTT_DEV_FWD_ORDER_BATCH=2" "TTT_DEV_FWD_ORDER_BATCH=4" "TTT_DEV_FWD_ORDER_BATCH=6" "TTT_DEV_FWD_ORDER_BATCH=8" "TTT_DEV_FWD_ORDER_BATCH=12" 2>&1 | tee gpurun_out/${T}_ab.txt
for ob in 4 32; do TTT_DEV_FWD_ORDER_BATCH=$ob python bench.py --config qwen235b --no-e2e --no-cpu --no-loss --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('qwen ob=$ob', round(d['ms_per_step'],3), {k[4:-7]: round(x,3) for k,x in d['kernels_ms_per_step'].items()})"; done
for ob in 4 32; do TTT_DEV_FWD_ORDER_BATCH=$ob python bench.py --config longctx --no-e2e --no-cpu --no-loss --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('longctx ob=$ob', round(d['ms_per_step'],3), {k[4:-7]: round(x,3) for k,x in d['kernels_ms_per_step'].items()})"; done
