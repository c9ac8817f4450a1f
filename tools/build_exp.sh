#!/bin/bash
# Experiment builds of libssbh_cuda.so (dev A/B only; the shipped build never defines these):
#   tools/build_exp.sh NAME "-DFLAG ..."  ->  build_exp/NAME/libssbh_cuda.so
# Run with SSBH_CUDA_LIB=build_exp/NAME/libssbh_cuda.so python tools/quick_time.py ...
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
out=build_exp/$name; mkdir -p $out
objs=""
for f in paper_2308_02856_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC -Iinclude $flags -c $f -o $out/$b.o &
  objs="$objs $out/$b.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libssbh_cuda.so $objs -lcudart
echo built $out/libssbh_cuda.so
