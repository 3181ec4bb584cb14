run() { python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu --no-e2e --shape $1 --mode sat --kernel skinny 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print(f\"v=$V {d['config']['M']}x{d['config']['N']}x{d['config']['K']} sat {d['ms_per_step']*1000:8.2f} us  {r['achieved']:8.1f} GB/s\")
"; }
for V in 0 1 4; do export NGEMM_SKINNY_VARIANT=$V
for m in 1 4 16; do for nk in 768x768 3072x768 768x3072 4096x1024; do run ${m}x${nk}; done; done; done
