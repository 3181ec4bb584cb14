#!/bin/bash
for cfg in 0 1 2 3; do for sp in 1 2 3; do for spec in 300x520x1100 256x256x2048 129x65x640 513x300x1024; do
  NGEMM_TC_CFG=$cfg NGEMM_TC_SPLITS=$sp timeout 60 python scripts/probe_kernels.py tcgen05 $spec 1 2>&1 | tail -1 | sed "s/^/cfg=$cfg sp=$sp /"
done; done; done
