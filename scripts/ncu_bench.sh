#!/bin/bash
# usage: scripts/ncu_bench.sh TAG "<bench args>" KERNEL_REGEX
# plain run first (must exit 0), then the launch list and one --set full capture of the top kernel.
TAG=$1; ARGS=$2; KRX=${3:-tc_gemm}
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > gpurun_out/ncu_list_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRX -s 1 -c 1 -o gpurun_out/prof_$TAG \
    python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/plain_$TAG.log
