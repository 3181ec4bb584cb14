#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
for spec in "simt 256x384x640 1" "simt 256x384x640 0" "skinny 8x768x768 1" "skinny 8x768x768 0" "tcgen05 128x256x128 1" "tcgen05 256x384x640 1" "tcgen05 1024x1024x1024 1"; do
  timeout 60 python scripts/probe_kernels.py $spec || echo "probe failed rc=$?: $spec"
done
