#!/bin/bash
# c5 (16384^3) raster group x L2 policy, interleaved twice on one box, 100 timed steps each.
for rep in 1 2; do for g in 4 8 16 32; do for h in 1 3; do
  NGEMM_TC_GROUP_M=$g NGEMM_TC_L2HINT=$h python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); c=d['clocks']
print('rep $rep group $g hint $h', d['value'], c['sm_mhz'], c['reasons'])"
  sleep 2
done; done; done
