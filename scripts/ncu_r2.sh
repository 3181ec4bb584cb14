#!/bin/bash
# Round 2: one --set full capture per kernel choice (each after its plain run exits 0) plus
# launch lists; run under gpurun (all ncu runs in one call count as one).  usage: ncu_r2.sh [tag ...]
set -u
mkdir -p gpurun_out
cap() {  # tag, bench args, kernel regex, launches to skip
  local tag=$1 args=$2 krx=$3 skip=${4:-2}
  python bench.py $args > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run failed: $tag"; return; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
      python bench.py $args > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$krx -s $skip -c 1 -o gpurun_out/prof_$tag \
      python bench.py $args > gpurun_out/ncu_full_$tag.log 2>&1
  echo "captured $tag rc=$?"
}
want() { [ $# -eq 0 ] && return 0; for t in "${TAGS[@]}"; do [ "$t" = "$1" ] && return 0; done; return 1; }
TAGS=("$@")
E="--steps 3 --warmup 2 --no-cpu --no-e2e --no-verify --no-sustained --no-shapes --eager"
want c5_tc        && cap c5_tc        "$E" tc_gemm
want c3_tc        && cap c3_tc        "$E --shape 2048x4096x1024" tc_gemm
want c4_tc        && cap c4_tc        "$E --shape 2048x2048x2048" tc_gemm
want c1_tc        && cap c1_tc        "$E --shape 1024x1024x1024" tc_gemm
want c2_mma       && cap c2_mma       "$E --shape 16x4096x1024" skinny_mma
want c2_sat       && cap c2_sat       "$E --shape 16x4096x1024 --mode sat" skinny_sat
want c4_satfix_ext && cap c4_satfix_ext "$E --shape 2048x2048x2048 --mode sat --adist max --bdist max" sat_fix
want c3_simt_sat  && cap c3_simt_sat  "$E --shape 128x4096x1024 --mode sat" simt_gemm
true
