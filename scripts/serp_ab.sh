#!/bin/bash
# 256x512 pair tiles: serpentine accumulator order over the K slabs (one accumulator change per stage) vs fixed order (two)
run() {
  local shape=$1; shift
  env "$@" timeout 300 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $shape "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} {sys.argv[2]} {d['value']:.0f} TOPS {d['ms_per_step']*1000:.2f} us verified={d.get('verified')} sm_mhz={d['clocks']['sm_mhz']}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-800:])
PY
}
NGEMM_TC_SERP=1 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "every_tile_config and 9" 2>&1 | tail -2
for rep in 1 2 3; do
for c in 0 1; do
  run 16384x16384x16384 NGEMM_TC_SERP=$c
  run 8192x8192x8192 NGEMM_TC_SERP=$c
done
done
