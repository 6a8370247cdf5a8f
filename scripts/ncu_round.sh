#!/bin/bash
# Launch list (gpu__time_duration per kernel) of a few cfg2 steps plus one full
# ncu capture of k_jacobian.  usage: scripts/ncu_round.sh TAG
TAG=${1:-x}
python scripts/prof_step.py cfg2 3 > gpurun_out/plain_$TAG.log 2>&1 || { cat gpurun_out/plain_$TAG.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/prof_step.py cfg2 3 > gpurun_out/ncul_$TAG.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_jacobian -s 3 -c 1 \
  -o gpurun_out/prof_$TAG python scripts/prof_step.py cfg2 3 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
