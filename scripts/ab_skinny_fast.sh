#!/bin/bash
# A/B (same box, interleaved): branch-free fast load path in the skinny kernels (NGEMM_SKINNY_FAST)
run() { python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --shape $1 --mode $2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"$1 $2 fast=$3 {d['ms_per_step']*1e3:8.3f} us\")
"; }
for rep in 1 2; do
for m in 1 4 16; do for nk in 768x768 3072x768 768x3072 4096x1024; do for mode in exact sat; do
  for f in 0 1; do NGEMM_SKINNY_FAST=$f run ${m}x${nk} $mode $f; done
done; done; done; done
