#!/bin/bash
# A/B: L2 prefetch before the PDL wait (NGEMM_L2_PREFETCH) on the c2 skinny and c3 medium shapes.
run() { python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu --no-e2e --shape $1 --mode $2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print(f\"{d['config']['M']}x{d['config']['N']}x{d['config']['K']} {d['config']['mode']:5s} {d['kernel']:8s} {d['ms_per_step']*1000:9.2f} us {d['value']:9.2f} TOPS  {r['bound']} {r['achieved']} {r['unit']} frac={r['frac']}\")
    elif 'Error' in l or 'error' in l: print(l.strip())
"; }
for pf in 0 1; do
  echo "== NGEMM_L2_PREFETCH=$pf"
  export NGEMM_L2_PREFETCH=$pf
  for m in 1 4 16; do for nk in 768x768 3072x768 768x3072 4096x1024; do run ${m}x${nk} exact; done; done
  for m in 1 16; do for nk in 3072x768 4096x1024; do run ${m}x${nk} sat; done; done
  for m in 128 512 2048; do for nk in 1024x1024 4096x1024 1024x4096; do run ${m}x${nk} exact; done; done
done
