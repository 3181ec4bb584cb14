#!/bin/bash
# HardwareSaturating below the hybrid's size rule: forced hybrid chain vs the dense SIMT kernel
run() { python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-shapes --no-sustained --shape $1 --mode sat --bdist $2 --kernel $3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print(f\"{d['config']['M']}x{d['config']['N']}x{d['config']['K']} sat $2 $3 {d['ms_per_step']*1000:9.2f} us verified={d.get('verified')}\")
" ; }
for shape in 128x1024x1024 128x4096x1024 128x1024x4096 512x1024x1024 256x4096x1024 1024x1024x1024 64x4096x1024; do
  for dist in uniform normal; do for kern in simt sat_hybrid; do run $shape $dist $kern; done; done
done
