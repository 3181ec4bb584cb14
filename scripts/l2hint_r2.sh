#!/bin/bash
# c5 16384^3 exact: L2 policy bits (1 A evict_last, 2 B evict_first, 4 C store evict_first),
# 20-step burst and 300-step power-capped runs, interleaved twice in one call
mkdir -p gpurun_out
for rep in 1 2; do
for h in 3 7 5 1 4 0; do
  NGEMM_TC_L2HINT=$h timeout 120 python bench.py --no-shapes --no-cpu --no-e2e --no-verify --steps 20 --warmup 3 > gpurun_out/h.log 2>&1
  python - $h <<'PY'
import json,sys
for l in open("gpurun_out/h.log"):
    if l.startswith("{"):
        d=json.loads(l); s=d.get("sustained",{})
        print(f"hint={sys.argv[1]} burst={d['value']:.0f} TOPS sustained300={s.get('value')} TOPS sus_mhz={s.get('clocks',{}).get('sm_mhz')} pw={s.get('clocks',{}).get('power_w_max')}")
PY
done
done
