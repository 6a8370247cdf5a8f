#!/bin/bash
# Apply time with parts of the kernel skipped (PDST_SKIP bit mask, profiling only):
# 1 volume, 2 CIP, 4 sides, 8 mass, 16 assembly, 32 boundary kernel, 64 tile fixup
for m in ${@:-0 1 2 8 16 3 27 31 63 127}; do
  echo "skip=$m $(PDST_SKIP=$m python scripts/time_kernels.py cfg2 2>&1 | grep -E 'apply' | tr '\n' ' ')"
done
