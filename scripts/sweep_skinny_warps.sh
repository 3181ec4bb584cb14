#!/bin/bash
# Skinny exact (warp-MMA stream): CTA width 8 / 16 / 32 warps (32 = one 1024-thread CTA per SM by
# registers, so N = 4096 takes two waves; 16 = two CTAs per SM).  Interleaved twice.
for rep in 1 2; do for s in 1x768x768 1x3072x768 1x768x3072 1x4096x1024 16x4096x1024 16x768x3072 4x3072x768; do
  for w in auto 8 16 32; do
    if [ $w = auto ]; then unset NGEMM_SKINNY_WARPS; else export NGEMM_SKINNY_WARPS=$w; fi
    python bench.py --shape $s --steps 50 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('rep $rep $s warps=$w', round(d['ms_per_step']*1000,2), 'us')"
  done
done; done
