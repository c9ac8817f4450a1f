cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_c3.csv python tools/quick_time.py --configs 3 --reps 1 > gpurun_out/ll_c3.log 2>&1
echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_f4 -s 2 -c 1 -o gpurun_out/leaf_c3 python tools/quick_time.py --configs 3 --reps 1 > gpurun_out/leaf_c3.log 2>&1
echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_tree -s 1 -c 1 -o gpurun_out/tree_c3 python tools/quick_time.py --configs 3 --reps 1 > gpurun_out/tree_c3.log 2>&1
echo rc=$?
