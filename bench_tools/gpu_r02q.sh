T=r02q
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
make variant VNAME=p1 EXTRA=-DTTT_FWD_PROBE=1 >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=p3 EXTRA=-DTTT_FWD_PROBE=3 >> gpurun_out/${T}_build.txt 2>&1
make variant VNAME=np3 EXTRA="-DTTT_FWD_PROBE=3 -DTTT_FWD_PERSIST=0" >> gpurun_out/${T}_build.txt 2>&1
for v in paper_2603_18567_b200/libtttattn.so build/libtttattn_p1.so build/libtttattn_p3.so build/libtttattn_np3.so build/libtttattn_prev.so; do
  TTT_ATTN_LIB=$v timeout 300 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/${T}_ab.json').read().strip().splitlines()[-1])
print('$v'.split('/')[-1], round(d['ms_per_step'],3), {k[4:-7]: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'fwd/step', [round(x,3) for x in d['per_ttt_step_ms']['fwd_ms']])
"
done
