#!/bin/bash
# Leaf-GEMM A/B on config 3: MMA-warp wait (SSBH_MMA_F4_SPIN 1 = poll, 0 = suspended; run as SSBH_MMA_SPIN before the f4 knob existed) and producer
# sets (SSBH_MMA_F4_SETS 2 | 3); one parity pass on the suspended wait first.
mkdir -p gpurun_out
SSBH_MMA_F4_SPIN=0 timeout 600 python -m pytest tests/test_tensor_engine.py tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1
for i in 1 2; do
  for v in "SSBH_MMA_F4_SPIN=1" "SSBH_MMA_F4_SPIN=0" "SSBH_MMA_F4_SETS=3" "SSBH_MMA_F4_SPIN=0 SSBH_MMA_F4_SETS=3"; do
    tag=$(echo $v | tr ' =' '__')
    env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_leaf_${tag}_$i.json 2>&1
    echo "$v run $i rc=$?"
  done
done
