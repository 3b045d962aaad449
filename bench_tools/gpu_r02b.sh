# r02b: fused forward diagonal + membar-free unroll pre-pass: tests, bench, A/B vs the separate diag kernel
T=r02b
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=nofuse EXTRA=-DTTT_FWD_FUSED_DIAG=0 >> gpurun_out/${T}_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_tree.py tests/test_gpu_edge_cases.py tests/test_gpu_bwd_unroll.py -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${T}_pytest_quick.txt
cat gpurun_out/${T}_pytest_quick.txt | tail -3
timeout 600 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --bwd-unroll --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_bench_unroll.json 2>&1
TTT_ATTN_LIB=build/libtttattn_nofuse.so timeout 600 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_bench_nofuse.json 2>&1
timeout 600 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_bench2.json 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/${T}_pytest.txt
tail -5 gpurun_out/${T}_pytest.txt
for f in bench bench_unroll bench_nofuse bench2; do python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/${T}_$f.json").read().strip().splitlines()[-1])
    print("$f", round(d["ms_per_step"],3), d["clocks"]["sm_mhz"], {k: round(v,3) for k,v in d["kernels_ms_per_step"].items()})
except Exception as e:
    print("$f", "ERR", e)
PY
done
