#!/bin/bash
# cmd_bench analogue + per-call overhead of the drop-in API on one GPU (gpurun helper).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
B=paper_2308_02856_b200/ssbh-b200
S=000000000000000000000000000000000000000000000000000000000000002a
tools/call_overhead > gpurun_out/call_overhead.csv 2>&1
for i in 1 2; do $B bench --sizes 20000000,40000000 --ns 16 --seed $S; done > gpurun_out/cmdbench.log 2>&1
for i in 1 2; do $B bench --sizes 100000000 --ns 20 --out-ratio 0.0004 --seed $S; done >> gpurun_out/cmdbench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cmdbench_launches.csv $B bench --sizes 100000000 --ns 20 --out-ratio 0.0004 --repeats 1 --seed $S > /dev/null 2>&1
echo done
