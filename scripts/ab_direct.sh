#!/bin/bash
# A/B (interleaved, one box): direct vector-store epilogue vs TMA-store epilogue (NGEMM_TC_DIRECT)
run() { python bench.py --steps 40 --warmup 5 --no-cpu --no-e2e --shape $1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"$1 direct=$2 {d['ms_per_step']*1e3:8.3f} us {d['value']:8.1f} TOPS\")
"; }
for rep in 1 2; do
for shape in 128x1024x1024 128x4096x1024 128x1024x4096 512x1024x1024 512x4096x1024 512x1024x4096 2048x1024x1024 2048x4096x1024 2048x1024x4096 1024x1024x1024 2048x2048x2048 1000x1000x1000; do
  for d in 0 1; do NGEMM_TC_DIRECT=$d run $shape $d; done
done; done
