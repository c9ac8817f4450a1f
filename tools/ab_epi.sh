#!/bin/bash
# A/B of the leaf GEMM's epilogue warps (SSBH_MMA_F4_EPI 4 | 8), config 3; parity on 8 first.
mkdir -p gpurun_out
SSBH_MMA_F4_EPI=8 timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -1
for i in 1 2; do
  for e in 4 8; do
    SSBH_MMA_F4_EPI=$e timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abe${e}_$i.json 2>&1; echo "epi $e run $i rc=$?"
  done
done
SSBH_MMA_F4_EPI=8 timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/abe8_c2.json 2>&1; echo c2 rc=$?
timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/abe4_c2.json 2>&1; echo c2 rc=$?
