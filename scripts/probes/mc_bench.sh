#!/bin/bash
for rep in 1 2; do for s in 1024x1024x1024 128x4096x1024 512x4096x1024 2048x4096x1024 2048x2048x2048 4096x4096x4096; do
  for cfg in auto 7 8; do
    if [ $cfg = auto ]; then unset NGEMM_TC_CFG; else export NGEMM_TC_CFG=$cfg; fi
    timeout 60 python bench.py --shape $s --steps 30 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('rep $rep $s cfg=$cfg', round(d['ms_per_step']*1000,2), 'us')"
  done
done; done
