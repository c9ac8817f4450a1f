#!/bin/bash
# A/B of the double-buffered epilogue TMEM loads (build with -DSSBH_F4_EPI_DB, SSBH_CUDA_LIB).
mkdir -p gpurun_out
L=$PWD/paper_2308_02856_b200
SSBH_CUDA_LIB=$L/libssbh_cuda_db.so timeout 600 python -m pytest tests/test_tensor_engine.py tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1
for i in 1 2; do
  for b in "" _db; do
    SSBH_CUDA_LIB=$L/libssbh_cuda$b.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abdb$b\_$i.json 2>&1; echo "build '$b' run $i rc=$?"
  done
done
