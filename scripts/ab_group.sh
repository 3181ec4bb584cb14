for st in 300 20; do for g in 4 6 8 10 12; do
  NGEMM_TC_GROUP_M=$g python bench.py --steps $st --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('group', $g, 'steps', $st, d['value'], c['sm_mhz'], c['reasons'])"
  sleep 3
done; done
