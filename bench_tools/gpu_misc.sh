timeout 900 python -m pytest tests/test_gpu_loss.py tests/test_gpu_head_parallel.py tests/test_gpu_autograd.py -x -q 2>&1 | tail -3
for r in 1 2; do for v in paper_2603_18567_b200/libtttattn.so build/libtttattn_noring.so; do TTT_ATTN_LIB=$v timeout 120 python bench_tools/time_loss.py; done; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['next_rows']))"
