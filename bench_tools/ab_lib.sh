# A/B of library builds on the headline bench (interleaved rounds): bash bench_tools/ab_lib.sh TAG ROUNDS lib1 lib2 ...
T=$1; R=$2; shift 2
for r in $(seq $R); do
  for v in "$@"; do
    TTT_ATTN_LIB=$v timeout 600 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_ab.json 2>/dev/null
    python -c "
import json,sys
d=json.loads(open('gpurun_out/${T}_ab.json').read().strip().splitlines()[-1])
print('$v'.split('/')[-1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k[4:-7]: round(v,3) for k,v in d['kernels_ms_per_step'].items()})
"
  done
done
