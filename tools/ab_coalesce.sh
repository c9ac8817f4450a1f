#!/bin/bash
# A/B of three builds of the leaf GEMM on config 3 (SSBH_CUDA_LIB): _ab = suspended MMA wait,
# _ab2 = + 4 loads per Hankel unit, default = + coalesced, swizzled y staging. Parity first.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
L=$PWD/paper_2308_02856_b200
for i in 1 2; do
  for b in _ab _ab2 ""; do
    SSBH_CUDA_LIB=$L/libssbh_cuda$b.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abc$b\_$i.json 2>&1; echo "build '$b' run $i rc=$?"
  done
done
timeout 600 python bench.py > gpurun_out/abc_c3_default.json 2> gpurun_out/abc_c3_default.err; echo c3 rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_f4 -s 3 -c 1 -o gpurun_out/leaf_coal_c3 $CMD > gpurun_out/ncu_coal.log 2>&1; echo ncu rc=$?
