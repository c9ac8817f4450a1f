#!/bin/bash
# Quick GPU check of a kernel change: tensor-engine + split parity tests, then per-phase times of
# configs 1-3 (tools/quick_time.py). -> gpurun_out/quick_gpu.log
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_tensor_engine.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/quick_time.py --configs 1,2,3 --reps 3 "$@" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    if 'ms_hash' in d: print('config', d['config'], 'hash', d['ms_hash'], 'total', d['ms_total'], 'gbit/s', d['gbit_s'])
    elif 'key_sha' in d: print('config', d['config'], 'sha', d['key_sha'])
"
} 2>&1 | tee gpurun_out/quick_gpu.log
