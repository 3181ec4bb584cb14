#!/bin/bash
# c5 16384^3 exact: tile configuration A/B (0 pair 256x256, 4 quad = two pairs sharing A by
# multicast, 1 1-CTA 128x256), 20-step bench, interleaved twice
for rep in 1 2; do
for cfg in 0 4 1; do
  NGEMM_TC_QUAD=1 NGEMM_TC_CFG=$cfg timeout 120 python bench.py --no-shapes --no-cpu --no-e2e --no-verify --no-sustained --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $cfg <<'PY'
import json,sys
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"cfg={sys.argv[1]} {d['value']:.0f} TOPS sm_mhz={d['clocks']['sm_mhz']} pw={d['clocks']['power_w_max']}")
PY
done
done
