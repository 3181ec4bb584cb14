#!/bin/bash
# e2e variants of the c5 headline: streaming-store staging copies vs plain memcpy
mkdir -p gpurun_out
for v in stream plain; do
  if [ $v = plain ]; then export NGEMM_COPY_PLAIN=1; fi
  timeout 300 python bench.py --no-shapes --no-cpu --no-sustained --no-verify --steps 5 > gpurun_out/e2e_$v.log 2>&1
  python - "$v" <<'PY'
import json,sys
for l in open(f"gpurun_out/e2e_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d=json.loads(l)["e2e"]; v=d["variants"]
        print(sys.argv[1], "pinned", d["ms_per_step"], "pageable", v["pageable"]["ms_per_step"], "resident", v["resident_weight"]["ms_per_step"])
PY
done
