#!/bin/bash
# c5 pair kernel with parts switched off (trace build only; results are wrong by design):
# dbg 1 = no C stores, 2 = no MMAs, 3 = neither (operand stream only); cfg 1 (1-CTA): 4 = no loads
export NGEMM_LIB=$PWD/paper_1910_00178_b200/lib/libngemm_cuda_trace.so
for rep in 1 2; do
for spec in "0 0" "0 1" "0 2" "0 3" "1 0" "1 4" "1 6"; do
  set -- $spec
  NGEMM_TC_CFG=$1 NGEMM_TC_DBG=$2 timeout 120 python bench.py --no-shapes --no-cpu --no-e2e --no-verify --no-sustained --steps 20 --warmup 3 > gpurun_out/d.log 2>&1
  python - $1 $2 <<'PY'
import json,sys
for l in open("gpurun_out/d.log"):
    if l.startswith("{"):
        d=json.loads(l); print(f"cfg={sys.argv[1]} dbg={sys.argv[2]} {d['ms_per_step']:.3f} ms {d['value']:.0f} TOPS-equiv sm={d['clocks']['sm_mhz']}")
PY
done
done
