#!/bin/bash
for g in 4 8 16 32 64; do
  NGEMM_TC_GROUP_M=$g python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('group_m', $g, d['value'], d['ms_per_step'])"
  sleep 2
done
for g in 8 16; do
  NGEMM_TC_GROUP_M=$g python bench.py --steps 300 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('long group_m', $g, d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
  sleep 2
done
