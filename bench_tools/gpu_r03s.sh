#!/bin/bash
# r03s: CTA schedule knobs (dev env overrides): bwd head split / order batch, fwd order batch
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=r03s
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -30 gpurun_out/${T}_build.txt; exit 1; }
bash bench_tools/ab_env.sh $T 2 "-" "TTT_DEV_BWD_HSPLIT=2" "TTT_DEV_BWD_ORDER_BATCH=1" "TTT_DEV_BWD_ORDER_BATCH=4" "TTT_DEV_BWD_ORDER_BATCH=16" "TTT_DEV_BWD_ORDER_BATCH=64" "TTT_DEV_FWD_ORDER_BATCH=1" "TTT_DEV_FWD_ORDER_BATCH=4" "TTT_DEV_FWD_ORDER_BATCH=16" "TTT_DEV_FWD_ORDER_BATCH=64" 2>&1 | tee gpurun_out/${T}_ab.txt
