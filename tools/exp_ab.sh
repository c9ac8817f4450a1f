#!/bin/bash
# A/B of experiment builds (tools/build_exp.sh) on config 3: per-phase CUDA-event times of the
# in-tree build and each named build, with the default split levels and with split_levels=7.
#   tools/exp_ab.sh [NAME ...] -> gpurun_out/exp_ab.log
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
out=gpurun_out/exp_ab.log; : > $out
for name in intree "$@"; do
  lib=""
  [ "$name" != intree ] && lib="SSBH_CUDA_LIB=build_exp/$name/libssbh_cuda.so"
  for ov in ""; do
    env $lib timeout 300 python tools/quick_time.py --configs 3 --reps 3 $ov 2>&1 | grep -v lop3_peak >> $out
  done
done
cat $out | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    if 'ms_hash' in d: print(d['win'][-40:], 'scatter', d['ms_scatter'], 'hash', d['ms_hash'], 'total', d['ms_total'])
    elif 'key_sha' in d: print(d['win'][-40:], 'sha', d['key_sha'])
"
