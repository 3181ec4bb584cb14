for rep in 1 2; do for pi in 0 1; do for sh in 1024x1024x1024 128x1024x1024 512x1024x4096 2048x1024x1024; do
  NGEMM_TC_PREISSUE=$pi python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --shape $sh | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('preissue', $pi, '$sh', round(d['ms_per_step']*1000,2), 'us')"
done; done; done
