#!/bin/bash
# 256x512 pair tiles (cfg 9, one accumulator over all 512 TMEM columns) vs 256x256 pairs (cfg 0):
# parity of cfg 9 first, then 20-step benches interleaved twice at several shapes and raster groups
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "every_tile_config" 2>&1 | tail -3
run() {  # shape cfg extra-env...
  local shape=$1 cfg=$2; shift 2
  env "$@" NGEMM_TC_CFG=$cfg timeout 300 python bench.py --shape $shape --no-shapes --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > gpurun_out/c.log 2>&1
  python - $shape $cfg "$*" <<'PY'
import json,sys
ok=False
for l in open("gpurun_out/c.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(f"shape={sys.argv[1]} cfg={sys.argv[2]} {sys.argv[3]} {d['value']:.0f} TOPS {d['ms_per_step']*1000:.1f} us verified={d.get('verified')} sm_mhz={d['clocks']['sm_mhz']}")
if not ok: print("FAILED", sys.argv[1:], open("gpurun_out/c.log").read()[-800:])
PY
}
for rep in 1 2; do
  for cfg in 0 9; do run 16384x16384x16384 $cfg X=1; done
  run 16384x16384x16384 9 NGEMM_TC_GROUP_M=16
  run 16384x16384x16384 9 NGEMM_TC_GROUP_M=4
  for cfg in 0 9; do run 8192x8192x8192 $cfg X=1; done
  for cfg in 0 9; do run 4096x4096x4096 $cfg X=1; done
done
