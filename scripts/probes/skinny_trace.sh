#!/bin/bash
# Build and run the skinny-kernel phase trace (B200).
set -e
cd "$(dirname "$0")"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/skinny_trace skinny_trace.cu
/tmp/skinny_trace "$@"
