#!/bin/bash
# A/B of the leaf GEMM's A-producer y path (SSBH_MMA_F4_REGY): parity first, then alternating
# config-3 bench runs, config 5 and one ncu capture of the leaf GEMM on the register path.
mkdir -p gpurun_out
SSBH_MMA_F4_REGY=1 timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
for i in 1 2; do
  for r in 0 1; do
    SSBH_MMA_F4_REGY=$r timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_c3_regy${r}_$i.json 2>&1
    echo "regy=$r run $i rc=$?"
  done
done
SSBH_MMA_F4_REGY=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ab_c5_regy1.json 2>&1; echo c5 rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
SSBH_MMA_F4_REGY=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_f4 -s 3 -c 1 -o gpurun_out/leaf_regy_c3 $CMD > gpurun_out/ncu_regy.log 2>&1; echo ncu rc=$?
