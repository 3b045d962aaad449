set -x
timeout 900 python -m pytest tests/test_gpu_loss.py -x -q 2>&1 | tail -15 > gpurun_out/loss_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/loss_smoke.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/loss_bench.json 2> gpurun_out/loss_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ttt_loss_kernel -s 1 -c 1 -o gpurun_out/loss_full python bench_tools/prof_loss.py > gpurun_out/loss_ncu.log 2>&1
cat gpurun_out/loss_pytest.txt gpurun_out/loss_smoke.txt; tail -c 1500 gpurun_out/loss_bench.json
