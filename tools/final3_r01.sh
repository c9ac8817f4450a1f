#!/bin/bash
# Final tree (split L = 6 at config 3 by default): suite, smoke, config 3 bench line x2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/f3_c3.json 2> gpurun_out/f3_c3.err; echo c3 rc=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/f3_c3b.json 2>&1; echo c3b rc=$?
