#!/bin/bash
# skinny K splits: cluster/DSMEM reduction (SKINNY_XRED=1, default) vs zeroed C + atomics (0)
run() {
  env NGEMM_SKINNY_XRED=$3 timeout 120 python bench.py --shape $1 --mode $2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-shapes --no-sustained > gpurun_out/c.log 2>&1
  python - "$@" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"{sys.argv[1]:>14s} {sys.argv[2]:5s} xred={sys.argv[3]} {d['ms_per_step']*1000:8.2f} us verified={d.get('verified')}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-600:])
PY
}
for rep in 1 2; do
for shape in 16x768x3072 16x256x16384 16x768x768 9x768x3072 16x1024x8192; do
  for mode in exact sat; do for x in 1 0; do run $shape $mode $x; done; done
done
done
