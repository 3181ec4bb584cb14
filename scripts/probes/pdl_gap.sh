#!/bin/bash
set -e
cd "$(dirname "$0")"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pdl_gap pdl_gap.cu -lcuda
/tmp/pdl_gap
