#!/bin/bash
# saturating skinny GEMMs with M = 8 / 5: dp4a stream (variant 4, default for M <= 8) vs warp MMAs + sparse fix (5)
run() {
  env NGEMM_SKINNY_VARIANT=$3 timeout 120 python bench.py --shape $1 --mode sat --bdist $2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-shapes --no-sustained > gpurun_out/c.log 2>&1
  python - "$@" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"{sys.argv[1]:>14s} B={sys.argv[2]:8s} variant={sys.argv[3]} {d['ms_per_step']*1000:8.2f} us verified={d.get('verified')}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-600:])
PY
}
for rep in 1 2; do
for shape in 8x4096x1024 8x768x768 8x3072x768 8x768x3072 5x4096x1024; do
  for dist in normal uniform; do for v in 4 5; do run $shape $dist $v; done; done
done
done
