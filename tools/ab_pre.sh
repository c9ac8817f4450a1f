#!/bin/bash
# A/B of the leaf GEMM's y prefetch depth (SSBH_F4_PRE build: 2 default vs 3), config 3.
mkdir -p gpurun_out
L=$PWD/paper_2308_02856_b200
SSBH_CUDA_LIB=$L/libssbh_cuda_p3.so timeout 600 python -m pytest tests/test_tensor_engine.py tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1
for i in 1 2; do
  for b in "" _p3; do
    SSBH_CUDA_LIB=$L/libssbh_cuda$b.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abp$b\_$i.json 2>&1; echo "build '$b' run $i rc=$?"
  done
done
