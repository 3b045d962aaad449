# A/B: programmatic dependent launch on / off (TTT_NO_PDL=1; the PDL build was reverted — kept as the record of the measurement)
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_bwd_bf16.py tests/test_gpu_bwd_unroll.py -x -q 2>&1 | tail -1
for r in 1 2 3; do
  for v in 0 1; do
    TTT_NO_PDL=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-loss | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('no_pdl=$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(sum(d['kernels_ms_per_step'].values()),3))"
  done
done
