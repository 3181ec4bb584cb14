#!/bin/bash
# A/B of the tcgen05 L2 policies at 16384^3 (bit 0: A evict_last, bit 1: B evict_first):
# throughput (20 and 100 steps) and per-launch DRAM bytes (ncu, metrics only).
for st in 20 100; do for rep in 1 2; do for h in 0 1 2 3; do
  NGEMM_TC_L2HINT=$h python bench.py --steps $st --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('l2hint', $h, 'steps', $st, d['value'], c['sm_mhz'], c['reasons'])"
  sleep 2
done; done; done
for h in 0 1 2 3; do
  NGEMM_TC_L2HINT=$h ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --eager 2>/dev/null \
     | grep -E "dram__bytes|gpu__time|hit_rate" | awk -F'","' -v h=$h '{print "l2hint", h, $(NF-2), $(NF-1), $NF}'
done
