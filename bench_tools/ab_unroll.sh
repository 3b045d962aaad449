# A/B: per-call backward vs one ttt_attn_bwd_unroll per unroll (whole-step bench, alternating)
timeout 900 python -m pytest tests/test_gpu_bwd_unroll.py tests/test_gpu_bwd_bf16.py -x -q 2>&1 | tail -1
for r in 1 2 3; do
  for m in "" "--bwd-unroll"; do
    timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-loss $m | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m' or 'per-call', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done
