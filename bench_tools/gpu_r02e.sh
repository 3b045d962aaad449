# r02e: ILP diagonal warps in the forward; A/B vs the separate diag kernel; bwd main pipeline trace
T=r02e
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=nofuse EXTRA=-DTTT_FWD_FUSED_DIAG=0 >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=trace EXTRA=-DTTT_TRACE >> gpurun_out/${T}_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fwd_bf16.py tests/test_gpu_edge_cases.py tests/test_gpu_ttt_length.py tests/test_gpu_tree.py -m gpu -x -q 2>&1 | tail -4
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_nofuse.so 2>&1 | tee gpurun_out/${T}_ab.txt
timeout 300 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_bench.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1])
print('fwd per step', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']], 'bwd per step', [round(x,3) for x in d['per_ttt_step_ms']['bwd_ms']])
"
for c in 0 40 300 700; do TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_bwd.py $c > gpurun_out/${T}_trace_cta$c.txt 2>&1; done
TTT_ATTN_LIB=build/libtttattn_trace.so timeout 120 python bench_tools/trace_bwd.py 40 timeline > gpurun_out/${T}_trace_timeline.txt 2>&1
head -40 gpurun_out/${T}_trace_cta40.txt
