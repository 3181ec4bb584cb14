python -m pytest tests -m gpu -x -q -k "every_tile_config" 2>&1 | tail -2
for cfg in auto 2 3 5 6; do
  echo "== cfg $cfg"
  if [ $cfg = auto ]; then python scripts/probes/tc_trace.py 128x1024x1024 512x4096x1024 1024x1024x1024 2048x2048x2048 2048x4096x1024;
  else NGEMM_TC_CFG=$cfg python scripts/probes/tc_trace.py 128x1024x1024 512x4096x1024 1024x1024x1024 2048x2048x2048 2048x4096x1024; fi
done
