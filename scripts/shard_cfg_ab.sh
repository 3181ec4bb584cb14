#!/bin/bash
# per-rank shard shapes of the 16384^3 GEMM (N = 8, 4, 2 GPUs): planner vs forced 256x256 pairs (0) / 256x512 tiles (9)
run() {
  local shape=$1; shift
  env "$@" timeout 300 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --no-verify --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $shape "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} {sys.argv[2]:18s} {d['value']:.0f} TOPS {d['ms_per_step']*1000:.2f} us")
if not ok: print("FAILED", sys.argv[1:])
PY
}
for rep in 1 2; do
for shape in 2048x16384x16384 4096x16384x16384 8192x16384x16384; do
  run $shape PLANNER=1
  run $shape NGEMM_TC_CFG=0
  run $shape NGEMM_TC_CFG=9
done
done
