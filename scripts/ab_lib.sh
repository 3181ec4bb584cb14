#!/bin/bash
# A/B of two in-tree builds (lib/libngemm_cuda_base.so vs lib/libngemm_cuda.so) on one box:
# ab_lib.sh "<bench args>" shape1 shape2 ...   (interleaved twice)
args=$1; shift
for rep in 1 2; do
for lib in base new; do
  if [ $lib = base ]; then export NGEMM_LIB=$PWD/paper_1910_00178_b200/lib/libngemm_cuda_base.so; else unset NGEMM_LIB; fi
  for s in "$@"; do
    timeout 120 python bench.py --shape $s $args --no-cpu --no-e2e --no-verify --no-sustained > gpurun_out/ab.log 2>&1
    python - $s $lib <<'PY'
import json,sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"{sys.argv[2]:5s} {sys.argv[1]:16s} {d['config']['mode']:5s} {d['ms_per_step']*1e3:9.2f} us  {d['kernel']}")
PY
  done
done
done
