for st in 20 300; do for h in 0 1 0 1; do for g in 8 16; do
  NGEMM_TC_L2HINT=$h NGEMM_TC_GROUP_M=$g python bench.py --steps $st --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('l2hint', $h, 'group', $g, 'steps', $st, d['value'], c['sm_mhz'], c['reasons'])"
  sleep 3
done; done; done
