#!/bin/bash
# Last session of round 1: full GPU suite on the default build, A/B of the B-producer load reuse
# (SSBH_CUDA_LIB = the build before it), then the default bench lines for configs 3 and 5.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
AB=paper_2308_02856_b200/libssbh_cuda_ab.so
for i in 1 2; do
  SSBH_CUDA_LIB=$PWD/$AB timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin_before_$i.json 2>&1; echo before $i rc=$?
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin_after_$i.json 2>&1; echo after $i rc=$?
done
timeout 600 python bench.py > gpurun_out/fin_c3.json 2> gpurun_out/fin_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/fin_c5.json 2>&1; echo c5 rc=$?
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/fin_c4.json 2>&1; echo c4 rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_f4 -s 3 -c 1 -o gpurun_out/leaf_fin_c3 $CMD > gpurun_out/ncu_fin.log 2>&1; echo ncu rc=$?
