#!/bin/bash
# c2 saturating shapes (sigma 32 B), graph-timed via bench --shape (L2-cold rotation)
for s in 16x4096x1024 16x768x3072 16x3072x768 16x768x768 4x4096x1024 4x768x3072 1x4096x1024 1x768x768; do
  timeout 120 python bench.py --shape $s --mode sat --steps 200 --warmup 5 --no-cpu --no-e2e --no-verify --no-sustained > gpurun_out/ss.log 2>&1
  python - $s <<'PY'
import json,sys
for l in open("gpurun_out/ss.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"{sys.argv[1]:14s} sat {d['ms_per_step']*1e3:8.2f} us  {d['kernel']}")
PY
done
