#!/bin/bash
# A/B of one library knob on one box: ab_knob.sh NAME "v1 v2 ..." "<bench args>" shape...  (interleaved twice)
name=$1; vals=$2; args=$3; shift 3
for rep in 1 2; do
for v in $vals; do
  for s in "$@"; do
    env NGEMM_$name=$v timeout 120 python bench.py --shape $s $args --no-cpu --no-e2e --no-verify --no-sustained > gpurun_out/ab.log 2>&1
    python - $s $name=$v <<'PY'
import json,sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"{sys.argv[2]:14s} {sys.argv[1]:18s} {d['config']['mode']:5s} {d['ms_per_step']*1e3:10.2f} us {d['value']:9.1f} TOPS {d['kernel']}")
PY
  done
done
done
