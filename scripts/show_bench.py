"""Pretty-print bench.py JSON lines (headline keys + the per-shape table)."""
import json
import sys

for path in sys.argv[1:]:
    for l in open(path):
        if not l.startswith('{'):
            print(l.rstrip()[:300])
            continue
        d = json.loads(l)
        sh = d.pop('shapes', None)
        print(json.dumps(d, indent=1)[:8000])
        for s in sh or []:
            if 'error' in s:
                print(s)
                continue
            r = s['roofline']
            print(f"{s['config']} {s['M']:>5}x{s['N']:>5}x{s['K']:>5} {s['mode']:5s} a={s['a'][:9]:9s} "
                  f"b={s['b'][:10]:10s} {s['kernel']:10s} {s['us']:9.2f}us {s['value']:8.2f} TOPS "
                  f"{r['bound']:6s} frac={r['frac']:.3f} v={s['verified']}")
