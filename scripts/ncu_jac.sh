#!/bin/bash
# One full ncu capture of k_jacobian at cfg2 (after a clean run of the same script).
# usage: scripts/ncu_jac.sh TAG
TAG=${1:-jac}
python scripts/time_kernels.py cfg2 > gpurun_out/plain_$TAG.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_jacobian -s 3 -c 1 \
  -o gpurun_out/prof_$TAG python scripts/time_kernels.py cfg2 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
