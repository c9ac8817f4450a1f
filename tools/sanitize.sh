#!/bin/bash
# compute-sanitizer, one tool per run, over tools/sanitize_cases.py (small shapes); logs to
# gpurun_out/sanitize_<tool>.log. racecheck/synccheck cover shared-memory hazards and barrier
# misuse in the warp-specialised mbarrier/TMEM pipelines; memcheck covers out-of-bounds access.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
done
