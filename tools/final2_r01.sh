#!/bin/bash
# Final bench lines on the final build (8 epilogue warps by default): suite, smoke, configs 3/1/2/5.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/f2_c3.json 2> gpurun_out/f2_c3.err; echo c3 rc=$?
for c in 1 2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f2_c$c.json 2>&1; echo c$c rc=$?; done
timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/f2_c5.json 2>&1; echo c5 rc=$?
