#!/bin/bash
# start stagger of the persistent units (TC_STAGGER = spread in ns) on the 256x512 pair tiles
run() {
  local shape=$1; shift
  env "$@" timeout 300 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --no-verify --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $shape "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} {sys.argv[2]} {d['value']:.0f} TOPS {d['ms_per_step']*1000:.1f} us sm_mhz={d['clocks']['sm_mhz']}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-800:])
PY
}
for rep in 1 2; do
for d in 0 4000 8000 16000 32000 64000; do
  run 16384x16384x16384 NGEMM_TC_STAGGER=$d
done
for d in 0 8000 32000; do
  run 8192x8192x8192 NGEMM_TC_STAGGER=$d
  run 16384x16384x16384 NGEMM_TC_STAGGER=$d NGEMM_TC_CFG=0
done
done
