#!/bin/bash
# c5 e2e (pinned) with the C tiles' D2H split into column strips of NGEMM_D2H_COLS
for rep in 1 2; do
for w in 0 1024 2048 4096; do
  if [ $w = 0 ]; then unset NGEMM_D2H_COLS; else export NGEMM_D2H_COLS=$w; fi
  timeout 300 python bench.py --no-shapes --no-cpu --no-sustained --no-verify --steps 5 > gpurun_out/e.log 2>&1
  python - $w <<'PY'
import json,sys
for l in open("gpurun_out/e.log"):
    if l.startswith("{"):
        d=json.loads(l)["e2e"]; v=d["variants"]
        print("strip", sys.argv[1], "pinned", d["ms_per_step"], "resident", v["resident_weight"]["ms_per_step"])
PY
done
done
