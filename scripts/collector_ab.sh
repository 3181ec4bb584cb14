#!/bin/bash
# 256x512 pair tiles: A-collector hints (first MMA of a K step fills, second reuses) vs plain MMAs
run() {
  local shape=$1; shift
  env "$@" timeout 300 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $shape "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} {sys.argv[2]} {d['value']:.0f} TOPS {d['ms_per_step']*1000:.2f} us verified={d.get('verified')} sm_mhz={d['clocks']['sm_mhz']}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-800:])
PY
}
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "every_tile_config and 9" 2>&1 | tail -2
NGEMM_TC_COLLECTOR=1 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "every_tile_config and 9" 2>&1 | tail -2
for rep in 1 2 3; do
for c in 0 1; do
  run 16384x16384x16384 NGEMM_TC_COLLECTOR=$c
  run 8192x8192x8192 NGEMM_TC_COLLECTOR=$c
done
done
for c in 0 1; do
NGEMM_TC_COLLECTOR=$c python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-shapes --no-sustained --no-verify | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['clocks']; print('collector', $c, 'steps 300', d['value'], d['ms_per_step'], c['sm_mhz'], c['power_w_max'], c['reasons'])"
sleep 3
done
