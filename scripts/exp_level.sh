#!/bin/bash
# Level-apply measurements at cfg5: the solve line, then the ncu list of the level kernels of one V-cycle.
mkdir -p gpurun_out
python bench.py --solve --config cfg5 > gpurun_out/solve_cfg5_now.json 2> gpurun_out/solve_cfg5_now.err
python scripts/prof_vcycle.py cfg5 5 > gpurun_out/prof_vcycle_now.log 2>&1
ncu -k regex:k_level --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/level_launches.csv python scripts/prof_vcycle.py cfg5 5 > gpurun_out/level_ncu.log 2>&1
tail -3 gpurun_out/prof_vcycle_now.log; head -c 600 gpurun_out/solve_cfg5_now.json
