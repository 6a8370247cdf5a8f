#!/bin/bash
# ncu --set full of the two patch inversion kernels (first launch of each) in the cfg5 solve's hierarchy build
mkdir -p gpurun_out
ncu -k regex:k_invert -c 2 --set full --clock-control none --import-source on -f -o gpurun_out/prof_invert python bench.py --solve --config cfg5 --max-krylov 2 > gpurun_out/prof_invert.log 2>&1
ls -la gpurun_out/prof_invert.ncu-rep
