#!/bin/bash
# raster group x L2 policy on the large square shapes (bench --shape, interleaved twice)
for rep in 1 2; do
for gm in 8 16 32; do
for h in 7 0; do
  for s in 4096x4096x4096 8192x8192x8192 16384x16384x16384; do
    st=100; [ $s = 16384x16384x16384 ] && st=20
    NGEMM_TC_GROUP_M=$gm NGEMM_TC_L2HINT=$h timeout 120 python bench.py --shape $s --steps $st --warmup 3 --no-cpu --no-e2e --no-verify --no-sustained > gpurun_out/ab.log 2>&1
    python - $s $gm $h <<'PY'
import json,sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"gm={sys.argv[2]:3s} hint={sys.argv[3]} {sys.argv[1]:18s} {d['ms_per_step']*1e3:10.2f} us {d['value']:8.1f} TOPS")
PY
  done
done
done
done
