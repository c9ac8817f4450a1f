#!/bin/bash
# A/B of the count-table geometry knobs at the config-4 and config-5 shapes (k = 64).
mkdir -p gpurun_out
for v in "7 16384" "4 65536" "3 131072"; do
  set -- $v
  SSBH_TABLE_BUDGET_SHIFT=$1 SSBH_MAX_CHUNKS=$2 timeout 600 python tools/sampler_time.py --log2n 34 --s 16384 --reps 2
  SSBH_TABLE_BUDGET_SHIFT=$1 SSBH_MAX_CHUNKS=$2 timeout 900 python tools/sampler_time.py --log2n 37 --s 32768 --chunks 8 --reps 1
done 2>&1 | tee gpurun_out/sampler_ab.log
