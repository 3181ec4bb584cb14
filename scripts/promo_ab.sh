#!/bin/bash
# L2 promotion of the operand tensor maps (TC_PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B = default)
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
for p in 3 2 1 0; do
  run 16384x16384x16384 NGEMM_TC_PROMO=$p
  run 16384x16384x16384 NGEMM_TC_PROMO=$p NGEMM_TC_CFG=0
  run 4096x4096x4096 NGEMM_TC_PROMO=$p
  run 2048x2048x2048 NGEMM_TC_PROMO=$p
done
done
