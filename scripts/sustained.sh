for g in 4 8 16 32; do
  NGEMM_TC_GROUP_M=$g python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('group_m', $g, 'steps 300', d['value'], d['ms_per_step'], c['sm_mhz'], c['power_w_max'], c['reasons'])"
  sleep 5
done
for st in 20 50 100; do
  python bench.py --steps $st --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('steps', $st, d['value'], d['ms_per_step'], c['sm_mhz'], c['power_w_max'], c['reasons'])"
  sleep 5
done
