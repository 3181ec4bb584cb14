for spec in 512x512x256 600x1024x700 1024x2048x2048 4096x4096x4096; do
  NGEMM_TC_CFG=4 timeout 60 python scripts/probe_kernels.py tcgen05 $spec 1 || echo "FAILED rc=$? $spec"
done
