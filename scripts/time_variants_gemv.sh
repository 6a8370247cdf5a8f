#!/bin/bash
echo "base $(python scripts/time_gemv.py 2>&1 | tr '\n' ' ')"
for f in exp/libpdst_*.so; do n=$(basename $f .so); echo "${n#libpdst_} $(PDST_LIB=$PWD/$f python scripts/time_gemv.py 2>&1 | tr '\n' ' ')"; done
