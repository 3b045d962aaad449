#!/bin/bash
# r02w: packed (cu_seqlens) batches — build, packed parity tests first, then the full GPU suite
# (padded-path regressions) and a short headline bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
make -j8 > gpurun_out/r02w_build.txt 2>&1 || { tail -30 gpurun_out/r02w_build.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_packed.py -x -q > gpurun_out/r02w_packed.txt 2>&1; echo "packed rc=$?" >> gpurun_out/r02w_packed.txt
tail -15 gpurun_out/r02w_packed.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02w_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02w_pytest.txt
tail -8 gpurun_out/r02w_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
python3 -c "
import json;d=json.load(open('gpurun_out/r02w_bench.json'));print(d['value'],d['ms_per_step'],d['kernels_ms_per_step'])" 
