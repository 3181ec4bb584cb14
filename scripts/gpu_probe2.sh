#!/bin/bash
for spec in "tcgen05 4096x2048x1024 1" "tcgen05 2200x2300x500 1" "tcgen05 2304x2304x384 1" "tcgen05 300x9000x1000 1"; do
  timeout 60 python scripts/probe_kernels.py $spec || echo "probe failed rc=$?: $spec"
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for cfg in 1 2; do NGEMM_TC_CFG=$cfg timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg', $cfg, d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done
