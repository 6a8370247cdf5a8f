#!/bin/bash
# launch list of the preconditioner build + full captures of its two heaviest kernels and of k_residual (cfg2)
mkdir -p gpurun_out
python scripts/time_build.py cfg2 > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_build.csv python scripts/time_build.py cfg2 > gpurun_out/ncu_build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_patch_fine -s 1 -c 1 -o gpurun_out/prof_patch_fine python scripts/time_build.py cfg2 >> gpurun_out/ncu_build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_invert_diag -s 1 -c 1 -o gpurun_out/prof_invert_diag python scripts/time_build.py cfg2 >> gpurun_out/ncu_build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_residual -s 2 -c 1 -o gpurun_out/prof_residual python scripts/time_residual.py cfg2 >> gpurun_out/ncu_build.log 2>&1
