#!/bin/bash
# e2e variants of the c5 headline: pinned staging slots per direction x host copy threads
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "4 7" "8 7" "8 11" "16 7"; do
  set -- $cfg
  NGEMM_STAGE_SLOTS=$1 NGEMM_COPY_THREADS=$2 timeout 300 python bench.py --no-shapes --no-cpu --no-sustained --no-verify --steps 5 > gpurun_out/e2e.log 2>&1
  python - "$1" "$2" <<'PY'
import json,sys
for l in open("gpurun_out/e2e.log"):
    if l.startswith("{"):
        d=json.loads(l)["e2e"]; v=d["variants"]
        print("slots", sys.argv[1], "threads", sys.argv[2], "pinned", d["ms_per_step"], "pageable", v["pageable"]["ms_per_step"], "resident", v["resident_weight"]["ms_per_step"])
PY
done
done
