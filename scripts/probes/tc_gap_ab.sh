#!/bin/bash
# Which tcgen05-kernel feature sets the ~2.3 us launch-to-launch gap?  (tc_trace, trace-build knobs;
# 1-CTA configs so that bit 2 applies)
S="1024x1024x1024 2048x4096x1024"
for cfg in 2 5; do
echo "== cfg $cfg default";                 NGEMM_TC_CFG=$cfg python scripts/probes/tc_trace.py $S
echo "== cfg $cfg no stores, no MMAs";      NGEMM_TC_CFG=$cfg NGEMM_TC_DBG=3 python scripts/probes/tc_trace.py $S
echo "== cfg $cfg no loads/MMAs/stores";    NGEMM_TC_CFG=$cfg NGEMM_TC_DBG=7 python scripts/probes/tc_trace.py $S
done
