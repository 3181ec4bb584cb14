#!/bin/bash
# Where the saturating hybrid chain's time goes on small shapes: skip launches one by one
# (NGEMM_SATFIX_SKIP bits: 1 prep A, 2 prep B, 8 tcgen05, 16 fix; results wrong).
for shape in ${SHAPES:-1024x1024x1024 512x1024x1024 2048x2048x2048}; do for dist in normal uniform; do
  for sk in 0 1 2 8 16 27; do
    NGEMM_SAT_HYBRID=1 NGEMM_SATFIX_SKIP=$sk python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --shape $shape --mode sat --bdist $dist 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"$shape $dist skip=$sk {d['ms_per_step']*1000:8.2f} us\")
"
  done
done; done
