#!/bin/bash
# tcgen05 tile configuration x split-K sweep on the c3 / c1 / c4 exact shapes (planner check).
run() { python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --shape $1 --kernel tcgen05 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print(f\"$1 cfg=$2 splits=$3 {d['ms_per_step']*1000:8.2f} us {d['value']:8.1f} TOPS {r['bound']} frac={r['frac']}\")
"; }
for shape in ${SHAPES:-128x1024x1024 128x4096x1024 128x1024x4096 512x1024x1024 512x4096x1024 512x1024x4096 2048x1024x1024 2048x4096x1024 2048x1024x4096 1024x1024x1024 2048x2048x2048}; do
  run $shape auto auto
  for cfg in 0 1 2 3; do for sp in 1 2 4; do
    NGEMM_TC_CFG=$cfg NGEMM_TC_SPLITS=$sp run $shape $cfg $sp
  done; done
done
