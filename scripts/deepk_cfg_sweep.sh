#!/bin/bash
# deep-K medium shapes: tile configuration x split-K sweep (graph-timed, L2-cold) next to the planner's choice
run() {
  local shape=$1; shift
  env "$@" timeout 120 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --no-verify --steps 100 --warmup 5 > gpurun_out/c.log 2>&1
  python - $shape "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} {sys.argv[2]:40s} {d['ms_per_step']*1000:8.2f} us")
if not ok: print("FAILED", sys.argv[1:])
PY
}
for shape in 2048x1024x4096 512x1024x4096 128x1024x4096 1024x1024x1024 2048x4096x1024; do
  run $shape PLANNER=1
  for cfg in 0 1 2 3; do for sp in 1 2 4 8; do run $shape NGEMM_TC_CFG=$cfg NGEMM_TC_SPLITS=$sp; done; done
done
