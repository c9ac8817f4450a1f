#!/bin/bash
# e2e A/B of the in-tree library against another build (build_exp/prev = the commit before a
# change, built with nvcc from `git archive`): config-3 bench lines under identical flags.
cd ${GRAFT_REPO_ROOT:-.}
p='import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],3), round(d["e2e"]["value"],3))'
for rep in 1 2; do
for lib in "" "SSBH_CUDA_LIB=build_exp/prev/libssbh_cuda.so"; do
  for fl in "--no-cpu-baseline" "--no-cpu-baseline --no-lop3-compare"; do
    echo -n "lib=[$lib] flags=[$fl]: "; env $lib timeout 600 python bench.py $fl 2>/dev/null | python -c "$p"
  done
done
done
