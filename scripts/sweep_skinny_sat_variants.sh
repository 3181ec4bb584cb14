#!/bin/bash
# sat skinny: rows-broadcast kernel (variant 1) vs dp4a load stream (variant 4) where the
# dispatcher currently picks the rows kernel (M > 4, N < 2048)
run() { python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --shape $1 --mode sat 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"$1 variant=$2 {d['ms_per_step']*1000:9.2f} us\")
"; }
for shape in 8x768x768 8x768x3072 8x1024x4096 16x768x768 16x768x3072 16x1024x1024 16x1536x768 12x768x768; do
  for v in 1 4; do NGEMM_SKINNY_VARIANT=$v run $shape $v; done
done
