#!/bin/bash
# Time the cfg2 apply with the in-tree library and every exp/libpdst_*.so variant.
echo "base $(python scripts/time_kernels.py cfg2 2>&1 | grep apply)"
for f in exp/libpdst_*.so; do
  n=$(basename $f .so); echo "${n#libpdst_} $(PDST_LIB=$PWD/$f python scripts/time_kernels.py cfg2 2>&1 | grep apply)"
done
