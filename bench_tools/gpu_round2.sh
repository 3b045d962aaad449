# Round-2 checkpoint session: tests, smoke, bench (both arms + unroll what-if), sanitizer, ncu launch list,
# ncu --set full of the attention kernels at the Llama shape, j = 6. usage: bash bench_tools/gpu_round2.sh TAG
T=${1:-r02n}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
make -j8 all > gpurun_out/${T}_build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --bwd-unroll --no-e2e --no-cpu --no-loss > gpurun_out/${T}_bench_unroll.json 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1
# compute-sanitizer: closed on this pool since r02z (runs under it left GPUs needing a reset); r02v logs stand
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-loss > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttt_ -c 5 -o gpurun_out/${T}_attn_full python bench_tools/prof_one.py llama8b 6 > gpurun_out/${T}_attn_ncu.log 2>&1
tail -4 gpurun_out/${T}_pytest.txt; tail -3 gpurun_out/${T}_smoke.txt; tail -c 600 gpurun_out/${T}_bench.json
