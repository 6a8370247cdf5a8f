#!/bin/bash
# ncu --set full of the level-1 Galerkin cell kernel and the coarse patch assembly in the cfg5 hierarchy build
mkdir -p gpurun_out
ncu -k regex:"k_galerkin_cells|k_patch_level" -c 2 --set full --clock-control none --import-source on -f -o gpurun_out/prof_build python bench.py --solve --config cfg5 --max-krylov 2 > gpurun_out/prof_build.log 2>&1
ls -la gpurun_out/prof_build.ncu-rep
