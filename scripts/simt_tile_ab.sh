#!/bin/bash
# SIMT saturating kernel: 128x128 tiles with K splits vs the default 64x64 plan
for rep in 1 2; do
for cfg in "-1 -1" "128 2" "128 4" "128 8"; do
  set -- $cfg
  for s in 128x4096x1024 128x1024x4096 512x1024x1024 256x2048x2048; do
    NGEMM_SIMT_TILE=$1 NGEMM_SIMT_SPLITS=$2 NGEMM_SAT_HYBRID=0 timeout 120 python bench.py --shape $s --mode sat --steps 50 --warmup 5 --no-cpu --no-e2e --no-verify --no-sustained > gpurun_out/ab.log 2>&1
    python - $s $1 $2 <<'PY'
import json,sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"tile={sys.argv[2]:4s} splits={sys.argv[3]:3s} {sys.argv[1]:16s} {d['ms_per_step']*1e3:8.2f} us {d['kernel']}")
PY
  done
done
done
