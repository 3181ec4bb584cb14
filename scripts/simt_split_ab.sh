#!/bin/bash
# SIMT saturating kernel on the small-M c3 shapes: split target (x SMs) x minimum split bytes
for rep in 1 2; do
for cfg in "2 512" "4 256" "6 256" "8 128"; do
  set -- $cfg
  for s in 128x1024x1024 128x4096x1024 128x1024x4096 512x1024x1024; do
    NGEMM_SKINNY_RG=$1 NGEMM_SKINNY_SPLITS=$2 timeout 120 python bench.py --shape $s --mode sat --steps 50 --warmup 5 --no-cpu --no-e2e --no-verify --no-sustained > gpurun_out/ab.log 2>&1
    python - $s $1 $2 <<'PY'
import json,sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"tgt={sys.argv[2]} min={sys.argv[3]:4s} {sys.argv[1]:16s} {d['ms_per_step']*1e3:8.2f} us {d['kernel']}")
PY
  done
done
done
