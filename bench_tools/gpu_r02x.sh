#!/bin/bash
# r02x: packed tests + smoke + A/B of the packed-capable library against the pre-packed build (headline)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
make -j8 > gpurun_out/r02x_build.txt 2>&1 || { tail -30 gpurun_out/r02x_build.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_packed.py -q > gpurun_out/r02x_packed.txt 2>&1; echo "packed rc=$?" >> gpurun_out/r02x_packed.txt
tail -4 gpurun_out/r02x_packed.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x_smoke.txt 2>&1; tail -3 gpurun_out/r02x_smoke.txt
bash bench_tools/ab_lib.sh r02x 3 build/ab/lib_prepacked.so paper_2603_18567_b200/libtttattn.so
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err
python3 -c "
import json;d=json.load(open('gpurun_out/r02x_bench.json'));print(json.dumps(d['next_rows']['packed']))"
