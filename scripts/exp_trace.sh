#!/bin/bash
mkdir -p gpurun_out
{ for f in exp/libpdst_trace*.so; do echo "== $f"; PDST_LIB=$PWD/$f python scripts/trace_apply.py ${1:-cfg2}; done; } > gpurun_out/exp_trace.log 2>&1
