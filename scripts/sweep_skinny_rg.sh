for rg in 1 2 4 8; do echo "== RG $rg"; NGEMM_SKINNY_RG=$rg PROBE_MODES=1 PROBE_G=1,128 timeout 300 python scripts/batched_probe.py; done
