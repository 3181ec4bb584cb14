python -m pytest tests -m gpu -x -q -k "skinny or batched or config2 or random or acceptance or leading or sat" > gpurun_out/t_sk.log 2>&1; tail -2 gpurun_out/t_sk.log
run() { python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --shape $1 --mode $2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print(f\"{d['config']['M']}x{d['config']['N']}x{d['config']['K']} {d['config']['mode']:5s} {d['kernel']:8s} {d['ms_per_step']*1000:9.2f} us {r['achieved']} {r['unit']} frac={r['frac']}\")
"; }
for m in 1 4 16; do for nk in 768x768 3072x768 768x3072 4096x1024; do run ${m}x${nk} sat; done; done
PROBE_MODES=0 PROBE_G=1,128 python scripts/batched_probe.py
