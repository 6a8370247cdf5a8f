#!/bin/bash
# A/B of the staggered phase order (in-tree) against exp/ variants; traces.
mkdir -p gpurun_out
{
python -m pytest tests/test_gpu_operator.py tests/test_gpu_vanka.py tests/test_gpu_partition.py -x -q -m gpu 2>&1 | tail -3
for i in 1 2; do
echo "base $(python scripts/time_kernels.py cfg2 2>&1 | grep -E 'apply|defect')"
for f in exp/libpdst_*.so; do
  case $f in *trace*) continue;; esac
  n=$(basename $f .so); echo "${n#libpdst_} $(PDST_LIB=$PWD/$f python scripts/time_kernels.py cfg2 2>&1 | grep -E 'apply|defect')"
done
done
for f in exp/libpdst_trace*.so; do echo "== $f"; PDST_LIB=$PWD/$f python scripts/trace_apply.py cfg2; done
echo "cfg3 base $(python scripts/time_kernels.py cfg3 2>&1 | grep -E 'apply')"
echo "cfg3 nostag $(PDST_LIB=$PWD/exp/libpdst_nostag.so python scripts/time_kernels.py cfg3 2>&1 | grep -E 'apply')"
} > gpurun_out/exp_stagger.log 2>&1
