#!/bin/bash
# 256x512 pair tiles at c5: raster group and L2 eviction hints (bit 0 A evict_last, bit 1 B evict_first, bit 2 C evict_first)
run() {
  local shape=$1; shift
  env "$@" timeout 300 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --no-verify --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $shape "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} {sys.argv[2]} {d['value']:.0f} TOPS {d['ms_per_step']*1000:.2f} us sm_mhz={d['clocks']['sm_mhz']}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-800:])
PY
}
for rep in 1 2; do
for g in 8 6 10 12; do run 16384x16384x16384 NGEMM_TC_GROUP_M=$g; done
for h in 7 3 5 1 6; do run 16384x16384x16384 NGEMM_TC_L2HINT=$h; done
done
