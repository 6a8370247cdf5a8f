#!/bin/bash
# Registers / spills of k_jacobian for a (possibly patched) copy of pdst_operator.cu: scripts/regs.sh [file]
F=${1:-/root/repo/paper_2603_28706_b200/csrc/pdst_operator.cu}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -Xcompiler -fPIC -Xptxas -v \
  -I/root/repo/paper_2603_28706_b200/csrc -I/root/repo/include -c -o /tmp/regs_$$.o "$F" 2>&1 | grep -E " error|k_jacobianILi[0-9]ELb" -A2 | grep -E "error|registers|spill" | paste - - | awk '{print $1,$2,$3,$4, $(NF-5), $(NF-4)}'
rm -f /tmp/regs_$$.o
