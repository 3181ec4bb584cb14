for st in 20 300; do for cfg in 0 4; do
  NGEMM_TC_CFG=$cfg python bench.py --steps $st --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('cfg', $cfg, 'steps', $st, d['value'], d['ms_per_step'], c['sm_mhz'], c['power_w_max'], c['reasons'])"
  sleep 5
done; done
