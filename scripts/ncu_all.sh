#!/bin/bash
# One --set full capture per kernel choice (each after its plain run exits 0), plus launch lists.
set -u
mkdir -p gpurun_out
cap() {  # tag, bench args, kernel regex
  local tag=$1 args=$2 krx=$3
  python bench.py $args > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run failed: $tag"; return; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
      python bench.py $args > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$krx -s 2 -c 1 -o gpurun_out/prof_$tag \
      python bench.py $args > gpurun_out/ncu_full_$tag.log 2>&1
  echo "captured $tag rc=$?"
}
cap c5_tc      "--steps 3 --warmup 2 --no-cpu --no-e2e --eager" tc_gemm
cap c1_tc      "--steps 3 --warmup 2 --no-cpu --no-e2e --eager --shape 1024x1024x1024" tc_gemm
cap c2_tcskinny "--steps 3 --warmup 2 --no-cpu --no-e2e --eager --shape 16x4096x1024" tc_skinny
cap c2_rows_sat "--steps 3 --warmup 2 --no-cpu --no-e2e --eager --shape 16x4096x1024 --mode sat" skinny_rows
cap c4_simt_sat "--steps 3 --warmup 2 --no-cpu --no-e2e --eager --shape 2048x2048x2048 --mode sat" simt_gemm
cap c3_tc      "--steps 3 --warmup 2 --no-cpu --no-e2e --eager --shape 2048x4096x1024" tc_gemm
