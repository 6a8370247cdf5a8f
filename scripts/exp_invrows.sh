#!/bin/bash
# register-resident exact inversion + k_invert_diag occupancy variant: parity, then build times
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_vanka.py tests/test_gpu_multigrid.py tests/test_gpu_cfg2_golden.py tests/test_gpu_solvers.py -m gpu -x -q > gpurun_out/invrows_tests.log 2>&1
tail -3 gpurun_out/invrows_tests.log
pick='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], "step_us %.1f" % (d["ms_per_step"]*1e3), "build_ms %.3f" % d["kernels"]["patch_build"]["ms"])'
for i in 1 2; do
python bench.py --no-cpu-baseline --no-secondary 2>/dev/null | python -c "$pick" cfg2-base
PDST_LIB=$PWD/exp/libpdst_lb4.so python bench.py --no-cpu-baseline --no-secondary 2>/dev/null | python -c "$pick" cfg2-lb4
done
python bench.py --no-cpu-baseline --no-secondary --config cfg5 2>/dev/null | python -c "$pick" cfg5-base
PDST_LIB=$PWD/exp/libpdst_lb4.so python bench.py --no-cpu-baseline --no-secondary --config cfg5 2>/dev/null | python -c "$pick" cfg5-lb4
python bench.py --solve --config cfg5 > gpurun_out/solve_invrows.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/solve_invrows.json'));print('solve build_s',d['preconditioner_build_s'],'vcycle',d['ms_per_vcycle'],'iters',d['krylov_iterations'])"
ncu -k regex:k_invert --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/invrows_ncu.csv python bench.py --solve --config cfg5 > /dev/null 2>&1
grep k_invert gpurun_out/invrows_ncu.csv | awk -F'","' '{print substr($5,1,40), $NF}' | head -12
