#!/bin/bash
# Config 4's extreme operands in saturating mode: hybrid chain vs the dense CUDA-core kernel.
for shape in 2048x2048x2048 1000x1000x1000; do for ab in "max max" "max min" "uniform max"; do
  set -- $ab
  for hy in 1 0; do
    NGEMM_SAT_HYBRID=$hy python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --shape $shape --mode sat --adist $1 --bdist $2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"$shape A=$1 B=$2 hybrid=$hy {d['ms_per_step']*1000:8.2f} us\")
"
  done
done; done
