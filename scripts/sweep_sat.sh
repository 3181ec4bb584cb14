run() { python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu --no-e2e --shape $1 --mode $2 ${3:+--kernel $3} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print(f\"{d['config']['M']}x{d['config']['N']}x{d['config']['K']} {d['config']['mode']:5s} {d['kernel']:8s} {d['ms_per_step']*1000:9.2f} us {d['value']:9.2f} TOPS\")
"; }
for shape in 1024x1024x1024 2048x2048x2048 1000x1000x1000 128x1024x1024 128x4096x1024 128x1024x4096 512x1024x1024 512x4096x1024 512x1024x4096 2048x1024x1024 2048x4096x1024 2048x1024x4096; do run $shape sat; done
for m in 1 4 16; do for nk in 768x768 3072x768 768x3072 4096x1024; do run ${m}x${nk} sat; done; done
