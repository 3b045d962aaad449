# r02c: L2-prefetched forward diagonal ring, fused dq conversion in the unroll backward, fp64 check-path
# accumulators, bench default = unroll backward; out_lo-free numerics probe
T=r02c
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_edge_cases.py tests/test_gpu_bwd_unroll.py tests/test_gpu_check_mode.py tests/test_gpu_ttt_length.py -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${T}_pytest_quick.txt
tail -3 gpurun_out/${T}_pytest_quick.txt
timeout 600 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --bwd-percall --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_bench_percall.json 2>&1
TTT_TEST_NO_OUTLO=1 timeout 900 python -m pytest tests/test_gpu_bwd_bf16.py tests/test_gpu_edge_cases.py -m gpu -q 2>&1 | tail -12 > gpurun_out/${T}_pytest_nolo.txt
tail -4 gpurun_out/${T}_pytest_nolo.txt
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt
tail -4 gpurun_out/${T}_pytest.txt
for f in bench bench_percall; do python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/${T}_$f.json").read().strip().splitlines()[-1])
    print("$f", round(d["ms_per_step"],3), d["clocks"]["sm_mhz"], {k: round(v,3) for k,v in d["kernels_ms_per_step"].items()}, [round(x,3) for x in d["per_ttt_step_ms"]["fwd_ms"]])
except Exception as e:
    print("$f", "ERR", e)
PY
done
