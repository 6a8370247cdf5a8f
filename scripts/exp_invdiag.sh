#!/bin/bash
# k_invert_diag change: parity tests that go through the diagonalized inverses, then the build time at cfg2 / cfg5.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vanka.py tests/test_gpu_multigrid.py tests/test_gpu_cfg2_golden.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/invdiag_tests.log 2>&1
tail -3 gpurun_out/invdiag_tests.log
pick='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], "step_us %.1f" % (d["ms_per_step"]*1e3), "build_ms %.3f" % d["kernels"]["patch_build"]["ms"])'
for i in 1 2; do python bench.py --no-cpu-baseline --no-secondary 2>/dev/null | python -c "$pick" cfg2; done
python bench.py --no-cpu-baseline --no-secondary --config cfg5 2>/dev/null | python -c "$pick" cfg5
ncu -k regex:k_invert_diag --metrics gpu__time_duration.sum --clock-control none -c 4 --csv --log-file gpurun_out/invdiag_ncu.csv python bench.py --no-cpu-baseline --no-secondary --config cfg5 --steps 2 --warmup 3 > /dev/null 2>&1
grep k_invert_diag gpurun_out/invdiag_ncu.csv | awk -F'","' '{print $5, $NF}' | head -4
