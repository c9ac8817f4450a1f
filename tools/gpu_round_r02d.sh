#!/bin/bash
# Round-2 final GPU session (after the windowed scatter): driver-style suite, smoke, bench lines (configs 3, 1, 2, 4, 5),
# reference arm, ncu launch list + full captures of the leaf GEMM, the sampler and the combine.
set -x
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c3.json 2>&1
for c in 1 2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>&1; done
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 rc=$?
timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-lop3-compare --e2e-steps 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_leaf_gemm -s 3 -c 1 -o gpurun_out/leaf_c3 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_count_ranked|k_scatter_windowed" -s 6 -c 2 -o gpurun_out/sampler_c3 $CMD > gpurun_out/ncu_sampler.log 2>&1; echo ncu4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_split_tree|k_hankel_units" -s 3 -c 2 -o gpurun_out/split_c3 $CMD > gpurun_out/ncu_split.log 2>&1; echo ncu5 rc=$?
ls -la gpurun_out
