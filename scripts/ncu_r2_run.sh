#!/bin/bash
# captures + on-box summaries (the .ncu-rep files are too big to bring back all at once)
bash scripts/ncu_r2.sh "$@" > gpurun_out/ncu_r2.log 2>&1
for t in "$@"; do
  NCU_OUT=gpurun_out NCU_SOURCE=1 python scripts/ncu_summary.py $t > /dev/null 2>&1 || echo "summary failed $t" >> gpurun_out/ncu_r2.log
  sz=$(stat -c %s gpurun_out/prof_$t.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 12000000 ]; then rm -f gpurun_out/prof_$t.ncu-rep; fi
done
rm -f gpurun_out/plain_*.log
du -sh gpurun_out >> gpurun_out/ncu_r2.log
