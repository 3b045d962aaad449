#!/bin/bash
# A/B of environment settings on the headline bench (interleaved rounds): bash bench_tools/ab_env.sh TAG ROUNDS "ENV1" "ENV2" ...
# each ENV is a space-separated list of VAR=value ("-" for none)
T=$1; R=$2; shift 2
for r in $(seq $R); do
  for v in "$@"; do
    envs=""; [ "$v" != "-" ] && envs="$v"
    env $envs timeout 600 python bench.py --no-e2e --no-cpu --no-loss --steps 20 > gpurun_out/${T}_abenv.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/${T}_abenv.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k[4:-7]: round(x,3) for k,x in d['kernels_ms_per_step'].items()})
"
  done
done
