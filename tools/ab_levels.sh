#!/bin/bash
# Final-tree check (suite + smoke) and the split-level A/B on config 3 after the epilogue change.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do
  for L in 5 6; do
    SSBH_MMA_SPLIT=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abl${L}_$i.json 2>&1; echo "L=$L run $i rc=$?"
  done
done
