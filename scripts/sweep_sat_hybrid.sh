#!/bin/bash
# HardwareSaturating, M > 16: hybrid dispatcher (tcgen05 on B_safe + sparse CUDA-core fix) vs the
# dense CUDA-core kernel, uniform B and config-2-like normal B (sigma 32).  Kernel times, one box.
run() { python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu --no-e2e --shape $1 --mode sat --bdist $2 ${3:+--kernel $3} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print(f\"{d['config']['M']}x{d['config']['N']}x{d['config']['K']} sat $2 {'$3' or 'auto':6s} {d['ms_per_step']*1000:9.2f} us {d['value']:9.2f} TOPS\")
" ; }
for shape in ${SHAPES:-1024x1024x1024 2048x2048x2048 1000x1000x1000 128x1024x1024 128x4096x1024 128x1024x4096 512x1024x1024 512x4096x1024 512x1024x4096 2048x1024x1024 2048x4096x1024 2048x1024x4096 4096x4096x4096}; do
  for dist in uniform normal; do run $shape $dist; done
  run $shape uniform simt
done
