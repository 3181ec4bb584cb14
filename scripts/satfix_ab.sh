#!/bin/bash
# saturating tensor-core + fix chain: base library vs new (stream-K fix kernel); bench --shape --mode sat
for rep in 1 2; do
for lib in base new; do
  if [ $lib = base ]; then export NGEMM_LIB=$PWD/paper_1910_00178_b200/lib/libngemm_cuda_base.so; else unset NGEMM_LIB; fi
  for spec in "2048x2048x2048 uniform uniform" "2048x2048x2048 max max" "1024x1024x1024 uniform uniform" "2048x4096x1024 uniform uniform" "512x4096x1024 uniform uniform" "1000x1000x1000 max min" "4096x4096x4096 uniform normal" "2048x2048x2048 uniform normal"; do
    set -- $spec
    timeout 120 python bench.py --shape $1 --mode sat --adist $2 --bdist $3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-verify --no-sustained > gpurun_out/ab.log 2>&1
    python - $lib "$spec" <<'PY'
import json,sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"{sys.argv[1]:5s} {sys.argv[2]:32s} {d['ms_per_step']*1e3:9.2f} us {d['kernel']}")
PY
  done
done
done
