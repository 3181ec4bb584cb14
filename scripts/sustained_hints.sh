#!/bin/bash
# 300-step (power-capped) runs of the 256x512 tiles under different L2 eviction hints / raster groups
for rep in 1 2; do
for env in "NGEMM_TC_L2HINT=7" "NGEMM_TC_L2HINT=5" "NGEMM_TC_L2HINT=3" "NGEMM_TC_L2HINT=0" "NGEMM_TC_GROUP_M=16" "NGEMM_TC_CFG=0"; do
  env $env python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-shapes --no-sustained --no-verify | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['clocks']; print('$env', 'steps 300', d['value'], d['ms_per_step'], c['sm_mhz'], c['power_w_max'], c['reasons'])"
  sleep 4
done
done
