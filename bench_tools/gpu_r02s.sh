T=r02s
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=wd EXTRA=-DTTT_WATCHDOG >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=np EXTRA=-DTTT_FWD_PERSIST=0 >> gpurun_out/${T}_build.txt 2>&1
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 180 python -m pytest tests/test_gpu_fwd_bf16.py -m gpu -q -x -k "small or determin" 2>&1 | tail -2
TTT_ATTN_LIB=build/libtttattn_wd.so timeout 120 python bench_tools/prof_one.py llama8b 6 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_tree.py tests/test_gpu_ttt_length.py tests/test_gpu_edge_cases.py tests/test_gpu_bwd_bf16.py -m gpu -q -x 2>&1 | tail -2
for v in paper_2603_18567_b200/libtttattn.so build/libtttattn_np.so build/libtttattn_prev.so paper_2603_18567_b200/libtttattn.so; do
  TTT_ATTN_LIB=$v timeout 300 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/${T}_ab.json').read().strip().splitlines()[-1])
print('$v'.split('/')[-1], round(d['ms_per_step'],3), {k[4:-7]: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'fwd/step', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])
"
done
