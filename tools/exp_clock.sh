cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for name in clock clock_noaprod clock_skel; do
 for ov in "" "--override split_levels=7"; do
  echo "== $name $ov"
  SSBH_CUDA_LIB=build_exp/$name/libssbh_cuda.so timeout 300 python tools/quick_time.py --configs 3 --reps 2 --f4-peak $ov 2>&1 | grep -E "EXPCLOCK|ms_hash|f4_peak" 
 done
done > gpurun_out/clk.log 2>&1
cat gpurun_out/clk.log
