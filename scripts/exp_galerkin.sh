#!/bin/bash
# Galerkin cell kernel change: multigrid parity, then the cfg5 hierarchy build and the kernel's ncu times
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/galerkin_tests.log 2>&1
tail -3 gpurun_out/galerkin_tests.log
python bench.py --solve --config cfg5 > gpurun_out/solve_galerkin.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/solve_galerkin.json'));print('solve build_s',d['preconditioner_build_s'],'vcycle',d['ms_per_vcycle'],'iters',d['krylov_iterations'],d['newton_message'])"
ncu -k regex:k_galerkin --metrics gpu__time_duration.sum --clock-control none -c 16 --csv --log-file gpurun_out/galerkin_ncu.csv python bench.py --solve --config cfg5 --max-krylov 2 > /dev/null 2>&1
grep k_galerkin gpurun_out/galerkin_ncu.csv | awk -F'","' '{print substr($5,1,40), $NF}' | head -16
