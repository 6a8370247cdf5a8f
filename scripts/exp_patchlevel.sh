#!/bin/bash
# k_patch_level: all Radau nodes per entry; parity, then ncu times (in-tree and the 2-CTA variant)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_solvers.py tests/test_gpu_dist_mg.py -m gpu -x -q > gpurun_out/patchlevel_tests.log 2>&1
tail -3 gpurun_out/patchlevel_tests.log
for v in base pl2; do
  if [ $v = base ]; then unset PDST_LIB; else export PDST_LIB=$PWD/exp/libpdst_$v.so; fi
  ncu -k regex:k_patch_level --metrics gpu__time_duration.sum --clock-control none -c 4 --csv --log-file gpurun_out/patchlevel_$v.csv python bench.py --solve --config cfg5 --max-krylov 2 > /dev/null 2>&1
  echo $v; grep k_patch_level gpurun_out/patchlevel_$v.csv | awk -F'","' '{print substr($5,1,40), $NF}' | head -4
done
