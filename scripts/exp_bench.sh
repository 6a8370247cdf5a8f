#!/bin/bash
# bench step time with the in-tree library and every exp/ variant
mkdir -p gpurun_out; : > gpurun_out/exp_bench.log
pick='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], "step_us %.1f" % (d["ms_per_step"]*1e3), "apply %.1f" % (d["roofline"]["launch_ms"]*1e3), "gemv %.1f" % (d["kernels"]["vanka_gemv"]["ms"]*1e3), "scatter %.1f" % (d["kernels"]["vanka_scatter"]["ms"]*1e3), "e2e %.2f" % d["e2e"]["value"])'
for i in 1 2; do
python bench.py --no-cpu-baseline --no-secondary 2>/dev/null | python -c "$pick" base >> gpurun_out/exp_bench.log
for f in exp/libpdst_*.so; do case $f in *trace*) continue;; esac
  n=$(basename $f .so); PDST_LIB=$PWD/$f python bench.py --no-cpu-baseline --no-secondary 2>/dev/null | python -c "$pick" ${n#libpdst_} >> gpurun_out/exp_bench.log
done; done
