#!/bin/bash
# One GPU session: tests, bench lines, reference arm, ncu launch list + full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4
# the other kernel paths on the same suite (plan overrides): the tiled kernel for every shared
# seed, and the LOP3 engine
timeout 900 python -m pytest tests -q -m gpu --ssbh-override shared_tiled=1 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_api.py -q -m gpu --ssbh-override engine=1 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench rc=$?
for c in 1 2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>&1; done
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1
timeout 1800 python bench.py --config 5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c3.json 2>&1
# launch list of the default bench command (tensor engine; the LOP3 comparison step is in it)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo ncu1 rc=$?
# the split's leaf GEMM (per step: remainder GEMM, then the leaf GEMM) and the direct tiled kernel
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_f4 -s 3 -c 1 -o gpurun_out/leaf_c3 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_mma_pb -s 3 -c 1 -o gpurun_out/mma_c3 $CMD --override split_levels=0 > gpurun_out/ncu_full_pb.log 2>&1; echo ncu2b rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_hash -c 1 -o gpurun_out/hash_c3 $CMD > gpurun_out/ncu_full_lop3.log 2>&1; echo ncu3 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_count_rows|k_scatter" -s 6 -c 2 -o gpurun_out/sampler_c3 $CMD > gpurun_out/ncu_sampler.log 2>&1; echo ncu4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split -s 3 -c 3 -o gpurun_out/split_c3 $CMD > gpurun_out/ncu_split.log 2>&1; echo ncu5 rc=$?
# config 5 launch list (one timed step after the warm-up; split leaf batches visible)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_list_c5.log 2>&1; echo ncu6 rc=$?
ls -la gpurun_out
