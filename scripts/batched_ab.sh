#!/bin/bash
# batched skinny probe: round-1 library vs current, same box, interleaved
for rep in 1 2; do
  NGEMM_LIB=$PWD/paper_1910_00178_b200/lib/libngemm_cuda_r1.so timeout 600 python scripts/batched_probe.py 2>&1 | grep -E "G= 128|G=   1" | sed "s/^/r1  /"
  timeout 600 python scripts/batched_probe.py 2>&1 | grep -E "G= 128|G=   1" | sed "s/^/new /"
done
