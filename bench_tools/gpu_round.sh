# Round-end style GPU session: tests, bench (both arms), launch list, ncu full of the loss kernel.
# usage: bash bench_tools/gpu_round.sh TAG
T=${1:-r01}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-loss > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ttt_loss_ring -s 1 -c 1 -o gpurun_out/${T}_loss_full python bench_tools/prof_loss.py > gpurun_out/${T}_loss_ncu.log 2>&1
cat gpurun_out/${T}_pytest.txt gpurun_out/${T}_smoke.txt | tail -8; tail -c 2500 gpurun_out/${T}_bench.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttt_ -c 5 -o gpurun_out/${T}_attn_full python bench_tools/prof_one.py llama8b 6 > gpurun_out/${T}_attn_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"ttt_fwd_sm100|ttt_qkv_rope_kernel" -c 2 -o gpurun_out/${T}_next_full python bench_tools/prof_next.py > gpurun_out/${T}_next_ncu.log 2>&1
