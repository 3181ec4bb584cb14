for shape in 16x768x768 16x3072x768 16x768x3072 16x4096x1024; do for sp in 1 2 4 8; do
  echo "== $shape splits=$sp"; NGEMM_SKINNY_SPLITS=$sp NGEMM_SKINNY_VARIANT=2 python scripts/latency_probe.py $shape 3 | tail -2
done; done
