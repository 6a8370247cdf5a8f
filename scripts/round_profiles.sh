#!/bin/bash
# Round evidence on one GPU: the bench line, the launch list of the same bench
# command (cold-cache, serialised: compare shares), per-launch DRAM traffic and
# one full capture of the apply kernel.  usage: scripts/round_profiles.sh TAG
TAG=${1:-r01}
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1 || { tail -5 gpurun_out/bench_$TAG.log; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1
python scripts/prof_step.py cfg2 3 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_jacobian -s 3 -c 1 \
  -o gpurun_out/prof_$TAG python scripts/prof_step.py cfg2 3 > gpurun_out/ncu_$TAG.log 2>&1
tail -c 300 gpurun_out/bench_$TAG.log
