timeout 600 python -m pytest tests/test_gpu_tree.py -x -q 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_fwd_bf16.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['next_rows']['tree_verify']))"
