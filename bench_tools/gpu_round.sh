set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r01c_pytest.txt
timeout 600 python bench.py > gpurun_out/r01c_bench.json 2> gpurun_out/r01c_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01c_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01c_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r01c_ncu_bench.log 2>&1
cat gpurun_out/r01c_pytest.txt gpurun_out/r01c_bench.json
