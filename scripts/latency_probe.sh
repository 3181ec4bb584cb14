for shape in 16x768x768 4x4096x1024 16x4096x1024 1x768x3072; do
  for v in 1 2; do for pdl in 1 0; do echo "== $shape variant=$v PDL=$pdl"; NGEMM_SKINNY_VARIANT=$v NGEMM_PDL=$pdl python scripts/latency_probe.py $shape 3; done; done
done
echo "== tcgen05 1024^3"; python scripts/latency_probe.py 1024x1024x1024 1; NGEMM_PDL=0 python scripts/latency_probe.py 1024x1024x1024 1
NGEMM_SKINNY_VARIANT=2 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e --shape 16x4096x1024 > /dev/null 2>&1 && NGEMM_SKINNY_VARIANT=2 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/launches_skinny.csv python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e --eager --shape 16x4096x1024 > /dev/null 2>&1; grep tc_skinny gpurun_out/launches_skinny.csv | tail -4
