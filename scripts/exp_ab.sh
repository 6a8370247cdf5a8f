#!/bin/bash
# A/B: in-tree library vs every exp/libpdst_*.so (no trace builds) at cfg2 (and cfg3 with CFG3=1)
mkdir -p gpurun_out
{
for i in 1 2; do
echo "base $(python scripts/time_kernels.py cfg2 2>&1 | grep -E 'apply|defect' | tr '\n' ' ')"
for f in exp/libpdst_*.so; do
  case $f in *trace*) continue;; esac
  n=$(basename $f .so); echo "${n#libpdst_} $(PDST_LIB=$PWD/$f python scripts/time_kernels.py cfg2 2>&1 | grep -E 'apply|defect' | tr '\n' ' ')"
done
done
if [ -n "$CFG3" ]; then
echo "cfg3 base $(python scripts/time_kernels.py cfg3 2>&1 | grep -E 'apply' | tr '\n' ' ')"
for f in exp/libpdst_*.so; do
  case $f in *trace*) continue;; esac
  n=$(basename $f .so); echo "cfg3 ${n#libpdst_} $(PDST_LIB=$PWD/$f python scripts/time_kernels.py cfg3 2>&1 | grep -E 'apply' | tr '\n' ' ')"
done
fi
} > gpurun_out/exp_ab.log 2>&1
if [ -n "$NCU" ]; then bash scripts/ncu_jac.sh $NCU; fi
