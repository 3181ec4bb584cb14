#!/bin/bash
# K sweep at M = N = 16384: time = waves x (K/128 x t_kb + E) -> per-K-slab time and the
# non-overlapped per-tile cost of 256x512 (cfg 9) vs 256x256 pairs (cfg 0)
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
for k in 1024 2048 4096 8192 16384; do
  for cfg in 0 9; do run 16384x16384x$k $cfg X=1; done
done
done
