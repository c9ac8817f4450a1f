#!/bin/bash
# Launch list (ncu gpu__time_duration) of one config-3 extraction for the in-tree build and each
# experiment build given: tools/exp_launches.sh [NAME ...] -> gpurun_out/exp_<name>.csv
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for name in intree "$@"; do
  lib=""
  [ "$name" != intree ] && lib="SSBH_CUDA_LIB=build_exp/$name/libssbh_cuda.so"
  env $lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/exp_$name.csv python tools/quick_time.py --configs 3 --reps 1 \
      > gpurun_out/exp_$name.log 2>&1
  echo "$name rc=$?"
done
