#!/bin/bash
# EXPERIMENT (timing only): operands read as if K-slab-major ([K/128][rows][128 B]; every TMA box one
# contiguous run) vs row-major boxes (128-byte pieces a row pitch apart). TC_TILED bit 0 = A, bit 1 = B.
run() {
  local shape=$1 cfg=$2; shift 2
  env "$@" NGEMM_TC_CFG=$cfg timeout 300 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --no-verify --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $shape $cfg "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} cfg={sys.argv[2]} {sys.argv[3]} {d['value']:.0f} TOPS {d['ms_per_step']*1000:.1f} us sm_mhz={d['clocks']['sm_mhz']}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-800:])
PY
}
for rep in 1 2; do
for cfg in 0 9; do
  for t in 0 1 2 3; do run 16384x16384x16384 $cfg NGEMM_TC_TILED=$t; done
done
for t in 0 3; do run 8192x8192x8192 9 NGEMM_TC_TILED=$t; run 4096x4096x4096 0 NGEMM_TC_TILED=$t; done
done
