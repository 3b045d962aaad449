# r02a: tests + bench + sanitizer + ncu of the backward pre-pass (unroll and per-call)
T=r02a
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
make -j8 all > gpurun_out/${T}_build.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/${T}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --bwd-unroll --no-e2e --no-cpu --no-loss > gpurun_out/${T}_bench_unroll.json 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1
timeout 1200 bash bench_tools/sanitize.sh $T > gpurun_out/${T}_sanitize_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ttt_bwd_pre -c 2 -o gpurun_out/${T}_pre_unroll python bench_tools/prof_unroll.py > gpurun_out/${T}_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ttt_bwd_pre|ttt_fwd_diag" -s 4 -c 2 -o gpurun_out/${T}_pre_percall python bench_tools/prof_one.py llama8b 6 > gpurun_out/${T}_ncu2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-loss > gpurun_out/${T}_ncu_bench.log 2>&1
cat gpurun_out/${T}_pytest.txt | tail -5; tail -c 1500 gpurun_out/${T}_bench.json; cat gpurun_out/${T}_sanitize_summary.txt | tail -25
