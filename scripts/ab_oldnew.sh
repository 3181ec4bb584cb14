#!/bin/bash
# same-box A/B: this tree vs ab_old/ (the previous session's final commit) on exact medium shapes
for rep in 1 2; do for s in 1024x1024x1024 2048x2048x2048 2048x4096x1024 16384x16384x16384; do
  st=30; [ $s = 16384x16384x16384 ] && st=20
  for tree in . ab_old; do
    (cd $tree && python bench.py --shape $s --steps $st --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('rep $rep $s tree=$tree', round(d['ms_per_step']*1000,2), 'us', d['value'], d['clocks']['sm_mhz'])")
  done
done; done
