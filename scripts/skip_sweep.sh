#!/bin/bash
# Apply time at cfg2 with parts of the kernel masked out (PDST_SKIP bits:
# 1 volume, 2 CIP, 4 boundary sides, 8 temporal mass, 16 node assembly).
for m in 0 1 2 4 8 16 3 31; do
  echo "skip=$m $(PDST_SKIP=$m python scripts/time_kernels.py cfg2 2>&1 | grep apply)"
done
